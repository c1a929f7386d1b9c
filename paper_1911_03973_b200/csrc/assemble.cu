// assemble.cu -- fused batched P1 element assembly (K_e, M_e, A_e, b_e) for triangles
// and tetrahedra.
//
// Triangles follow elements.py:56-137 operation by operation, so
// with -fmad=false the outputs are bit-identical to build_element_batch:
//   det = d1x*d2y - d1y*d2x;  area = 0.5*det;  gx_j = (y_jn - y_jp)/det;
//   gy_j = (x_jp - x_jn)/det;  K_ij = (gx_i*gx_j + gy_i*gy_j)*area;  M_ij = area*P_ij;
//   A = K + nu*M;  b_j = (f*area)/3.
// Tetrahedra follow the oracle restatement (oracle/ebs_oracle.py _geometry): cofactor
// gradients g_k = (d_{k+1} x d_{k+2})/det, g_0 = -((g_1+g_2)+g_3), vol = det/6.
//
// One thread per element; the element-major outputs (nb*nb doubles per element) are
// staged through shared memory so every global store is a coalesced, contiguous run.
#include "ebs_internal.cuh"

namespace ebs {

constexpr double EPS_AREA = 1e-14;    // elements.py:19
constexpr double EPS_VOLUME = 1e-18;  // oracle restatement

template <int NB>
__device__ __forceinline__ void stage_store(double (&v)[NB * NB], double *smem,
                                            double *__restrict__ out, int64_t e0,
                                            int64_t n_e) {
    constexpr int NB2 = NB * NB, STR = NB2 | 1;  // odd stride: no bank conflicts
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NB2; ++q) smem[threadIdx.x * STR + q] = v[q];
    __syncthreads();
    const int nel = (n_e - e0) < (int64_t)blockDim.x ? (int)(n_e - e0) : (int)blockDim.x;
    const int total = nel * NB2;
    double *dst = out + e0 * NB2;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int el = t / NB2, q = t - el * NB2;  // 32-bit: a block's run is < 2^31
        dst[t] = smem[el * STR + q];
    }
}

template <int NB>
__global__ void __launch_bounds__(128)
    k_assemble(int64_t n_e, const double *__restrict__ nodes, const int32_t *__restrict__ conn,
               double nu, const double *__restrict__ f_vals, double f_const,
               double *__restrict__ K_out, double *__restrict__ M_out, double *__restrict__ A_out,
               double *__restrict__ b_out, int64_t *n_degenerate) {
    constexpr int DIM = NB - 1, NB2 = NB * NB;
    extern __shared__ double smem[];
    const int64_t e0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t e = e0 + threadIdx.x;
    const bool valid = e < n_e;
    double K[NB2], M[NB2], A[NB2];
    double meas = 0.0;
    if (valid) {
        double p[NB][DIM];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            int64_t v = conn[j * n_e + e];
#pragma unroll
            for (int a = 0; a < DIM; ++a) p[j][a] = nodes[v * DIM + a];
        }
        double g[DIM][NB];
        if constexpr (NB == 3) {
            double d1x = p[1][0] - p[0][0], d1y = p[1][1] - p[0][1];
            double d2x = p[2][0] - p[0][0], d2y = p[2][1] - p[0][1];
            double det = d1x * d2y - d1y * d2x;
            meas = 0.5 * det;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int jn = (j + 1) % 3, jp = (j + 2) % 3;
                g[0][j] = (p[jn][1] - p[jp][1]) / det;
                g[1][j] = (p[jp][0] - p[jn][0]) / det;
            }
        } else {
            double d[3][3];
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int a = 0; a < 3; ++a) d[q][a] = p[q + 1][a] - p[0][a];
            // c23 = d2 x d3, c31 = d3 x d1, c12 = d1 x d2 (oracle _cross)
            double c[3][3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double *u = d[(k + 1) % 3], *w = d[(k + 2) % 3];
                c[k][0] = u[1] * w[2] - u[2] * w[1];
                c[k][1] = u[2] * w[0] - u[0] * w[2];
                c[k][2] = u[0] * w[1] - u[1] * w[0];
            }
            double det = (d[0][0] * c[0][0] + d[0][1] * c[0][1]) + d[0][2] * c[0][2];
            meas = det / 6.0;
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int a = 0; a < 3; ++a) g[a][k + 1] = c[k][a] / det;
#pragma unroll
            for (int a = 0; a < 3; ++a) g[a][0] = -((g[a][1] + g[a][2]) + g[a][3]);
        }
        const double eps = NB == 3 ? EPS_AREA : EPS_VOLUME;
        if (!(meas > eps)) atomicAdd((unsigned long long *)n_degenerate, 1ull);
        // _MASS_PATTERN = (ones + eye)/12 (elements.py:22); tets (ones + eye)/20
        const double pd = NB == 3 ? 2.0 / 12.0 : 2.0 / 20.0;
        const double po = NB == 3 ? 1.0 / 12.0 : 1.0 / 20.0;
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                double k = g[0][i] * g[0][j];
#pragma unroll
                for (int a = 1; a < DIM; ++a) k = k + g[a][i] * g[a][j];
                k = k * meas;
                double m = meas * (i == j ? pd : po);
                K[i * NB + j] = k;
                M[i * NB + j] = m;
                A[i * NB + j] = k + nu * m;
            }
        if (b_out) {
            double f = f_vals ? f_vals[e] : f_const;
            double bj = (f * meas) / (double)NB;
#pragma unroll
            for (int j = 0; j < NB; ++j) b_out[j * n_e + e] = bj;
        }
    } else {
#pragma unroll
        for (int q = 0; q < NB2; ++q) K[q] = M[q] = A[q] = 0.0;
    }
    if (K_out) stage_store<NB>(K, smem, K_out, e0, n_e);
    if (M_out) stage_store<NB>(M, smem, M_out, e0, n_e);
    if (A_out) stage_store<NB>(A, smem, A_out, e0, n_e);
}

__global__ void k_combine(int64_t count, const double *__restrict__ K,
                          const double *__restrict__ M, double nu, double *__restrict__ A) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        A[i] = K[i] + nu * M[i];  // elements.py:121
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_assemble_p1(int dim, int64_t n_e, const double *nodes, const int32_t *conn,
                    double nu, const double *f_vals, double f_const, double *K_e,
                    double *M_e, double *A_e, double *b_e, int64_t *n_degenerate,
                    void *stream) {
    EBS_TRY
    EBS_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3, got %d", dim);
    EBS_REQUIRE(nu >= 0.0, "nu must be nonnegative, got %g", nu);
    EBS_REQUIRE(n_degenerate, "n_degenerate must be a device int64 pointer");
    CU(cudaMemsetAsync(n_degenerate, 0, sizeof(int64_t), S(stream)));
    if (n_e == 0) return EBS_OK;
    const int block = 128;  // 256 measured slower (0.85 vs 0.97 of peak, 2D)
    const int64_t grid = (n_e + block - 1) / block;
    EBS_REQUIRE(grid < (1ll << 31), "too many elements");
    if (dim == 2) {
        size_t sm = block * (9 | 1) * sizeof(double);
        k_assemble<3><<<(unsigned)grid, block, sm, S(stream)>>>(
            n_e, nodes, conn, nu, f_vals, f_const, K_e, M_e, A_e, b_e, n_degenerate);
    } else {
        size_t sm = block * (16 | 1) * sizeof(double);
        k_assemble<4><<<(unsigned)grid, block, sm, S(stream)>>>(
            n_e, nodes, conn, nu, f_vals, f_const, K_e, M_e, A_e, b_e, n_degenerate);
    }
    LAUNCHED();
    EBS_CATCH
}

int ebs_combine(int64_t count, const double *K_e, const double *M_e, double nu, double *A_e,
                void *stream) {
    EBS_TRY
    EBS_REQUIRE(nu >= 0.0, "nu must be nonnegative, got %g", nu);
    if (count == 0) return EBS_OK;
    k_combine<<<grid_for(count, 256), 256, 0, S(stream)>>>(count, K_e, M_e, nu, A_e);
    LAUNCHED();
    EBS_CATCH
}

}  // extern "C"

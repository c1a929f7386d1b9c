// mesh.cu -- structured mesh generation, boundary detection, validation, relabelling.
//
// 2D follows mesh.py:104-148 (build_grid_mesh, _detect_boundary) bit for bit: the
// coordinates are the IEEE quotients i/(n-1) exactly as np.arange(n)/(n-1).
// 3D is the Kuhn-cube restatement of oracle/ebs_oracle.py:kuhn_cube_mesh.
#include "ebs_internal.cuh"

namespace ebs {

__global__ void k_grid2d_nodes(int64_t n, double *__restrict__ nodes) {
    const int64_t nn = n * n;
    const double den = (double)(n - 1);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nn;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t iy = k / n, ix = k - iy * n;
        nodes[2 * k] = (double)ix / den;
        nodes[2 * k + 1] = (double)iy / den;
    }
}

__global__ void k_grid2d_conn(int64_t n, int32_t *__restrict__ conn) {
    const int64_t nc = (n - 1) * (n - 1), n_e = 2 * nc;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
         c += (int64_t)gridDim.x * blockDim.x) {
        int64_t iy = c / (n - 1), ix = c - iy * (n - 1);
        int32_t ll = (int32_t)(iy * n + ix);
        int64_t e = 2 * c;
        // lower (ll, ll+1, ll+n+1), then upper (ll, ll+n+1, ll+n)   mesh.py:118-121
        conn[e] = ll;
        conn[n_e + e] = ll + 1;
        conn[2 * n_e + e] = ll + (int32_t)n + 1;
        conn[e + 1] = ll;
        conn[n_e + e + 1] = ll + (int32_t)n + 1;
        conn[2 * n_e + e + 1] = ll + (int32_t)n;
    }
}

__global__ void k_kuhn_nodes(int64_t N, double *__restrict__ nodes) {
    const int64_t n = N + 1, nn = n * n * n;
    const double den = (double)(n - 1);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nn;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix = k % n, t = k / n, iy = t % n, iz = t / n;
        nodes[3 * k] = (double)ix / den;
        nodes[3 * k + 1] = (double)iy / den;
        nodes[3 * k + 2] = (double)iz / den;
    }
}

__global__ void k_kuhn_conn(int64_t N, int32_t *__restrict__ conn) {
    // KUHN_PERMS = (012)(021)(102)(120)(201)(210); odd ones swap local vertices 2,3
    const int P0[6] = {0, 0, 1, 1, 2, 2}, P1[6] = {1, 2, 0, 2, 0, 1};
    const bool ODD[6] = {false, true, true, false, false, true};
    const int64_t n = N + 1, ncube = N * N * N, n_e = 6 * ncube;
    const int32_t step[3] = {1, (int32_t)n, (int32_t)(n * n)};
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncube;
         c += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix = c % N, t = c / N, iy = t % N, iz = t / N;
        int32_t v0 = (int32_t)((iz * n + iy) * n + ix);
        int32_t v3 = v0 + 1 + step[1] + step[2];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            int32_t v1 = v0 + step[P0[q]];
            int32_t v2 = v1 + step[P1[q]];
            int32_t a2 = ODD[q] ? v3 : v2, a3 = ODD[q] ? v2 : v3;
            int64_t e = 6 * c + q;
            conn[e] = v0;
            conn[n_e + e] = v1;
            conn[2 * n_e + e] = a2;
            conn[3 * n_e + e] = a3;
        }
    }
}

__global__ void k_flags(int dim, int64_t n_n, const double *__restrict__ nodes, int which,
                        uint8_t *__restrict__ flags) {
    const double tol = 1e-12;  // mesh.py:22 _BOUNDARY_TOL
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_n;
         k += (int64_t)gridDim.x * blockDim.x) {
        bool on = false;
        if (which == 0) {
            for (int a = 0; a < dim; ++a) {
                double v = nodes[k * dim + a];
                on |= (fabs(v) <= tol) | (fabs(v - 1.0) <= tol);
            }
        } else {
            on = fabs(nodes[k * dim + (dim - 1)]) <= tol;
        }
        flags[k] = on ? 1 : 0;
    }
}

__device__ __forceinline__ double measure_of(int dim, const double *__restrict__ nodes,
                                             const int32_t *v) {
    if (dim == 2) {
        double x0 = nodes[2 * (int64_t)v[0]], y0 = nodes[2 * (int64_t)v[0] + 1];
        double d1x = nodes[2 * (int64_t)v[1]] - x0, d1y = nodes[2 * (int64_t)v[1] + 1] - y0;
        double d2x = nodes[2 * (int64_t)v[2]] - x0, d2y = nodes[2 * (int64_t)v[2] + 1] - y0;
        return 0.5 * (d1x * d2y - d1y * d2x);  // mesh.py:96-101
    }
    double p0[3], d[3][3];
    for (int a = 0; a < 3; ++a) p0[a] = nodes[3 * (int64_t)v[0] + a];
    for (int q = 0; q < 3; ++q)
        for (int a = 0; a < 3; ++a) d[q][a] = nodes[3 * (int64_t)v[q + 1] + a] - p0[a];
    double cx = d[1][1] * d[2][2] - d[1][2] * d[2][1];
    double cy = d[1][2] * d[2][0] - d[1][0] * d[2][2];
    double cz = d[1][0] * d[2][1] - d[1][1] * d[2][0];
    return ((d[0][0] * cx + d[0][1] * cy) + d[0][2] * cz) / 6.0;
}

__global__ void k_check(int dim, int64_t n_n, int64_t n_e, const double *__restrict__ nodes,
                        const int32_t *__restrict__ conn, int64_t *counts) {
    const int nb = dim + 1;
    int64_t bad_idx = 0, bad_meas = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t v[4];
        bool ok = true;
        for (int j = 0; j < nb; ++j) {
            v[j] = conn[j * n_e + e];
            if (v[j] < 0 || v[j] >= n_n) { ok = false; ++bad_idx; }
        }
        if (ok && !(measure_of(dim, nodes, v) > 0.0)) ++bad_meas;
    }
    if (bad_idx) atomicAdd((unsigned long long *)&counts[0], (unsigned long long)bad_idx);
    if (bad_meas) atomicAdd((unsigned long long *)&counts[1], (unsigned long long)bad_meas);
}

__global__ void k_measure(int dim, int64_t n_e, const double *__restrict__ nodes,
                          const int32_t *__restrict__ conn, double *__restrict__ out) {
    const int nb = dim + 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t v[4];
        for (int j = 0; j < nb; ++j) v[j] = conn[j * n_e + e];
        out[e] = measure_of(dim, nodes, v);
    }
}

__global__ void k_permute(int dim, int64_t n_n, int64_t n_e, const int64_t *__restrict__ perm,
                          const double *__restrict__ nodes, const int32_t *__restrict__ conn,
                          double *__restrict__ nodes_out, int32_t *__restrict__ conn_out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < n_n; i += stride) {
        int64_t to = perm[i];
        for (int a = 0; a < dim; ++a) nodes_out[to * dim + a] = nodes[i * dim + a];
    }
    const int64_t nc = (int64_t)(dim + 1) * n_e;
    for (int64_t k = t0; k < nc; k += stride) conn_out[k] = (int32_t)perm[conn[k]];
}

__global__ void k_centroids(int dim, int64_t n_e, const double *__restrict__ nodes,
                            const int32_t *__restrict__ conn, double *__restrict__ out) {
    const int nb = dim + 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
         e += (int64_t)gridDim.x * blockDim.x) {
        for (int a = 0; a < dim; ++a) {
            double s = nodes[(int64_t)conn[e] * dim + a] + nodes[(int64_t)conn[n_e + e] * dim + a];
            for (int j = 2; j < nb; ++j) s = s + nodes[(int64_t)conn[j * n_e + e] * dim + a];
            out[e * dim + a] = s / (double)nb;  // elements.py:107 p.mean(axis=1)
        }
    }
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_mesh_grid2d(int64_t n, double *nodes, int32_t *conn, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 2, "need at least 2 nodes per side, got n=%lld", (long long)n);
    EBS_REQUIRE(n * n < (int64_t)ID_MASK, "mesh too large for int32 node ids");
    k_grid2d_nodes<<<grid_for(n * n, 256), 256, 0, S(stream)>>>(n, nodes);
    LAUNCHED();
    if (n > 1) {
        k_grid2d_conn<<<grid_for((n - 1) * (n - 1), 256), 256, 0, S(stream)>>>(n, conn);
        LAUNCHED();
    }
    EBS_CATCH
}

int ebs_mesh_kuhn3d(int64_t N, double *nodes, int32_t *conn, void *stream) {
    EBS_TRY
    EBS_REQUIRE(N >= 1, "need at least 1 cell per side, got N=%lld", (long long)N);
    EBS_REQUIRE((N + 1) * (N + 1) * (N + 1) < (int64_t)ID_MASK, "mesh too large");
    k_kuhn_nodes<<<grid_for((N + 1) * (N + 1) * (N + 1), 256), 256, 0, S(stream)>>>(N, nodes);
    LAUNCHED();
    k_kuhn_conn<<<grid_for(N * N * N, 128), 128, 0, S(stream)>>>(N, conn);
    LAUNCHED();
    EBS_CATCH
}

int ebs_mesh_flags(int dim, int64_t n_n, const double *nodes, int which, uint8_t *flags,
                   void *stream) {
    EBS_TRY
    EBS_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
    EBS_REQUIRE(which == 0 || which == 1, "which must be 0 or 1");
    if (n_n == 0) return EBS_OK;
    k_flags<<<grid_for(n_n, 256), 256, 0, S(stream)>>>(dim, n_n, nodes, which, flags);
    LAUNCHED();
    EBS_CATCH
}

int ebs_mesh_check(int dim, int64_t n_n, int64_t n_e, const double *nodes,
                   const int32_t *conn, int64_t *counts, void *stream) {
    EBS_TRY
    EBS_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
    CU(cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), S(stream)));
    if (n_e == 0) return EBS_OK;
    k_check<<<grid_for(n_e, 256), 256, 0, S(stream)>>>(dim, n_n, n_e, nodes, conn, counts);
    LAUNCHED();
    EBS_CATCH
}

int ebs_mesh_measure(int dim, int64_t n_e, const double *nodes, const int32_t *conn,
                     double *measure, void *stream) {
    EBS_TRY
    EBS_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
    if (n_e == 0) return EBS_OK;
    k_measure<<<grid_for(n_e, 256), 256, 0, S(stream)>>>(dim, n_e, nodes, conn, measure);
    LAUNCHED();
    EBS_CATCH
}

int ebs_mesh_permute(int dim, int64_t n_n, int64_t n_e, const int64_t *perm,
                     const double *nodes, const int32_t *conn, double *nodes_out,
                     int32_t *conn_out, void *stream) {
    EBS_TRY
    EBS_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
    int64_t work = n_n > (dim + 1) * n_e ? n_n : (dim + 1) * n_e;
    if (work == 0) return EBS_OK;
    k_permute<<<grid_for(work, 256), 256, 0, S(stream)>>>(dim, n_n, n_e, perm, nodes, conn,
                                                         nodes_out, conn_out);
    LAUNCHED();
    EBS_CATCH
}

int ebs_centroids(int dim, int64_t n_e, const double *nodes, const int32_t *conn,
                  double *out, void *stream) {
    EBS_TRY
    EBS_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
    if (n_e == 0) return EBS_OK;
    k_centroids<<<grid_for(n_e, 256), 256, 0, S(stream)>>>(dim, n_e, nodes, conn, out);
    LAUNCHED();
    EBS_CATCH
}

}  // extern "C"

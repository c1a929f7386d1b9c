// Microbenchmark: the C2 caller -> internal permutation y[m] = x[o2n[m]] (4.2M random 8 B
// reads from an L2-resident vector) through (a) the LSU path (ILP-8 gather, as
// k_to_internal_ilp) and (b) TMA tile::gather4 (x viewed as an (n/4, 4) f64 tensor: each
// gather4 fetches four 32 B rows straight from L2 into shared memory, bypassing the L1tex
// wavefront pipeline that bounds (a)).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_gather_probe scripts/tma_gather_probe.cu -lcuda
//   ./tma_gather_probe [n]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

constexpr int ILP = 8;

template <int IL>
__global__ void __launch_bounds__(256) k_lsu_t(int n, const int *__restrict__ o2n,
                                               const double *__restrict__ x, double *__restrict__ y) {
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * IL) {
        int idx[IL];
        double v[IL];
#pragma unroll
        for (int u = 0; u < IL; ++u) {
            const int m = base + u * stride;
            idx[u] = m < n ? __ldcs(o2n + m) : 0;
        }
#pragma unroll
        for (int u = 0; u < IL; ++u) {
            const int m = base + u * stride;
            v[u] = m < n ? __ldg(x + idx[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < IL; ++u) {
            const int m = base + u * stride;
            if (m < n) __stcs(y + m, v[u]);
        }
    }
}

__global__ void __launch_bounds__(256) k_lsu(int n, const int *__restrict__ o2n,
                                             const double *__restrict__ x, double *__restrict__ y) {
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * ILP) {
        int idx[ILP];
        double v[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int m = base + u * stride;
            idx[u] = m < n ? __ldcs(o2n + m) : 0;
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int m = base + u * stride;
            v[u] = m < n ? __ldg(x + idx[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int m = base + u * stride;
            if (m < n) y[m] = v[u];
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// one warp = one pipeline of S stages; a stage = 128 nodes = 32 gather4 (one per lane)
template <int S, int W>
__global__ void __launch_bounds__(W * 32) k_tma(const __grid_constant__ CUtensorMap tm, int n,
                                                const int *__restrict__ o2n,
                                                double *__restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[W][S];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double *ring = reinterpret_cast<double *>(smem) + (size_t)wib * S * 512;  // 128 rows x 4
    uint64_t *bar = bars[wib];
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int warp = blockIdx.x * W + wib, nwarps = gridDim.x * W;
    const int nst = (n + 127) / 128;  // stages of 128 nodes
    int idx_keep[S][4];
    auto issue = [&](int st, int slot) {
        const int base = st * 128 + lane * 4;
        int r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int m = base + q;
            const int id = m < n ? __ldcs(o2n + m) : 0;
            idx_keep[slot][q] = id;
            r[q] = id >> 2;
        }
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&bar[slot])),
                         "r"(128 * 32)
                         : "memory");
        __syncwarp();
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(ring + slot * 512 + lane * 16)),
            "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
            "r"(smem_u32(&bar[slot]))
            : "memory");
    };
    uint32_t phase = 0;
    int k = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int st = warp + s * nwarps;
        if (st < nst) issue(st, s);
    }
    for (int st = warp; st < nst; st += nwarps, ++k) {
        const int slot = k % S;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar[slot])),
            "r"((phase >> slot) & 1u)
            : "memory");
        phase ^= 1u << slot;
        const double *rs = ring + slot * 512 + lane * 16;
        const int base = st * 128 + lane * 4;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = rs[q * 4 + (idx_keep[slot][q] & 3)];
        __syncwarp();
        if (base + 3 < n) {
            reinterpret_cast<double2 *>(y + base)[0] = make_double2(v[0], v[1]);
            reinterpret_cast<double2 *>(y + base)[1] = make_double2(v[2], v[3]);
        } else {
            for (int q = 0; q < 4; ++q)
                if (base + q < n) y[base + q] = v[q];
        }
        const int nxt = st + S * nwarps;
        if (nxt < nst) issue(nxt, slot);
    }
}

// Hybrid: in each CTA, WL warps gather nodes [0, split) through the LSU (ILP-8), WT warps
// gather [split, n) through TMA gather4 (S-stage ring per warp) -- the two paths have
// separate throughput limits (L1tex wavefronts vs the TMA unit).
template <int S, int WL, int WT>
__global__ void __launch_bounds__((WL + WT) * 32) k_hyb(const __grid_constant__ CUtensorMap tm, int n,
                                                        int split, const int *__restrict__ o2n,
                                                        const double *__restrict__ x,
                                                        double *__restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[WT > 0 ? WT : 1][S];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (wib < WL) {
        const int stride = gridDim.x * WL * 32;
        for (int base = blockIdx.x * WL * 32 + threadIdx.x; base < split; base += stride * ILP) {
            int idx[ILP];
            double v[ILP];
#pragma unroll
            for (int u = 0; u < ILP; ++u) {
                const int m = base + u * stride;
                idx[u] = m < split ? __ldcs(o2n + m) : 0;
            }
#pragma unroll
            for (int u = 0; u < ILP; ++u) {
                const int m = base + u * stride;
                v[u] = m < split ? __ldg(x + idx[u]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < ILP; ++u) {
                const int m = base + u * stride;
                if (m < split) y[m] = v[u];
            }
        }
        return;
    }
    if constexpr (WT > 0) {
    const int tw = wib - WL;
    double *ring = reinterpret_cast<double *>(smem) + (size_t)tw * S * 512;
    uint64_t *bar = bars[tw];
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int warp = blockIdx.x * WT + tw, nwarps = gridDim.x * WT;
    const int nst = (n - split + 127) / 128;
    int idx_keep[S][4];
    auto issue = [&](int st, int slot) {
        const int base = split + st * 128 + lane * 4;
        int r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int m = base + q;
            const int id = m < n ? __ldcs(o2n + m) : 0;
            idx_keep[slot][q] = id;
            r[q] = id >> 2;
        }
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&bar[slot])),
                         "r"(128 * 32)
                         : "memory");
        __syncwarp();
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(ring + slot * 512 + lane * 16)),
            "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
            "r"(smem_u32(&bar[slot]))
            : "memory");
    };
    uint32_t phase = 0;
    int k = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int st = warp + s * nwarps;
        if (st < nst) issue(st, s);
    }
    for (int st = warp; st < nst; st += nwarps, ++k) {
        const int slot = k % S;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar[slot])),
            "r"((phase >> slot) & 1u)
            : "memory");
        phase ^= 1u << slot;
        const double *rs = ring + slot * 512 + lane * 16;
        const int base = split + st * 128 + lane * 4;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = rs[q * 4 + (idx_keep[slot][q] & 3)];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (base + q < n) y[base + q] = v[q];
        const int nxt = st + S * nwarps;
        if (nxt < nst) issue(nxt, slot);
    }
    }
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 4198401;
    const int n2 = (n + 3) / 4 * 4;
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::mt19937 rng(1);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<double> hx(n2);
    for (int i = 0; i < n2; ++i) hx[i] = 0.5 + i;
    int *o2n;
    double *x, *y;
    CK(cudaMalloc(&o2n, sizeof(int) * n));
    CK(cudaMalloc(&x, sizeof(double) * n2));
    CK(cudaMalloc(&y, sizeof(double) * n));
    CK(cudaMemcpy(o2n, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x, hx.data(), sizeof(double) * n2, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {4, (cuuint64_t)(n2 / 4)};
    cuuint64_t gstr[1] = {32};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstr, box,
                                         es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        printf("cuTensorMapEncodeTiled failed %d\n", (int)cr);
        return 1;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const bool flush = getenv("FLUSH") && atoi(getenv("FLUSH"));
    const size_t fbytes = 512ull << 20;
    void *fbuf = nullptr;
    if (flush) CK(cudaMalloc(&fbuf, fbytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto check = [&](const char *what) {
        std::vector<double> hy(n);
        CK(cudaMemcpy(hy.data(), y, sizeof(double) * n, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n; ++i)
            if (hy[i] != hx[perm[i]]) {
                printf("%s: mismatch at %d\n", what, i);
                return;
            }
    };
    auto timeit = [&](const char *what, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        CK(cudaMemset(y, 0, sizeof(double) * n));
        launch();
        CK(cudaDeviceSynchronize());
        check(what);
        const int R = 50;
        float ms = 0;
        if (flush) {
            std::vector<float> t;
            for (int i = 0; i < R; ++i) {
                CK(cudaMemsetAsync(fbuf, i & 0xff, fbytes));
                CK(cudaEventRecord(e0));
                launch();
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float m1 = 0;
                CK(cudaEventElapsedTime(&m1, e0, e1));
                t.push_back(m1);
            }
            std::sort(t.begin(), t.end());
            ms = t[R / 2] * R;
        } else {
            CK(cudaEventRecord(e0));
            for (int i = 0; i < R; ++i) launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
        }
        printf("%-28s %8.2f us%s\n", what, ms / R * 1e3, flush ? " (x flushed from L2, median)" : "");
    };
    timeit("lsu ilp8 8 CTA/SM", [&] {
        k_lsu<<<sms * 8, 256>>>(n, o2n, x, y);
    });
#define LSU_CASE(IL_, B_)                                                                 \
    {                                                                                     \
        char name[64];                                                                    \
        snprintf(name, sizeof name, "lsu ilp%d %d CTA/SM", IL_, B_);                      \
        timeit(name, [&] { k_lsu_t<IL_><<<sms * B_, 256>>>(n, o2n, x, y); });             \
    }
    LSU_CASE(4, 8) LSU_CASE(8, 8) LSU_CASE(16, 8) LSU_CASE(8, 4) LSU_CASE(16, 4) LSU_CASE(4, 16)
    LSU_CASE(8, 16) LSU_CASE(32, 2) LSU_CASE(16, 2)
    if (argc > 2 && argv[2][0] == 'q') return 0;
#define HYB_CASE(S_, WL_, WT_, B_, F_)                                                   \
    {                                                                                     \
        auto kern = k_hyb<S_, WL_, WT_>;                                                  \
        const size_t sm = (size_t)(WT_ > 0 ? WT_ : 1) * S_ * 512 * 8;                     \
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        const int split = (int)((long long)n * F_ / 100) / 128 * 128;                     \
        char name[64];                                                                    \
        snprintf(name, sizeof name, "hyb S=%d L%d T%d %d/SM f=%d%%", S_, WL_, WT_, B_, F_); \
        timeit(name, [&] { kern<<<sms * B_, (WL_ + WT_) * 32, sm>>>(tm, n, split, o2n, x, y); }); \
    }
    HYB_CASE(2, 8, 0, 6, 100)
    HYB_CASE(2, 8, 2, 5, 85) HYB_CASE(2, 8, 2, 5, 75) HYB_CASE(2, 8, 2, 5, 65)
    HYB_CASE(2, 8, 4, 4, 75) HYB_CASE(2, 8, 4, 4, 65) HYB_CASE(2, 8, 4, 4, 55)
    HYB_CASE(3, 8, 4, 4, 65) HYB_CASE(2, 6, 4, 4, 60) HYB_CASE(2, 8, 8, 3, 55)
    HYB_CASE(2, 8, 8, 3, 45) HYB_CASE(2, 4, 4, 6, 60)
    if (argc > 2) return 0;
#define TMA_CASE(S_, W_, B_)                                                              \
    {                                                                                     \
        auto kern = k_tma<S_, W_>;                                                        \
        const size_t sm = (size_t)W_ * S_ * 512 * 8;                                      \
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        char name[64];                                                                    \
        snprintf(name, sizeof name, "tma S=%d W=%d %d CTA/SM", S_, W_, B_);               \
        timeit(name, [&] { kern<<<sms * B_, W_ * 32, sm>>>(tm, n, o2n, y); });           \
    }
    TMA_CASE(2, 4, 4)
    TMA_CASE(4, 4, 4)
    TMA_CASE(4, 8, 4)
    TMA_CASE(8, 4, 4)
    TMA_CASE(4, 8, 8)
    TMA_CASE(8, 8, 4)
    TMA_CASE(2, 8, 8)
    return 0;
}

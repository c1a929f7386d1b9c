// sell.cuh -- the element-operator hot loop: node-centric, ordered, SELL-32 streaming.
//
// For internal node m (lane l of chunk c = m/32) the slots k = 0..cnt[m)-1 hold, in the
// reference bincount order j*n_e + e (operators.py:98), one contribution each:
//     loc = ((A[j,0]*x_0 + A[j,1]*x_1) + A[j,2]*x_2) [+ A[j,3]*x_3]   (operators.py:69 einsum)
// where x_i is the value at local vertex i of element e, and the node's sum runs
//     s = ((0.0 + c_0) + c_1) + ...                                      (np.bincount)
// with c_k = loc (matvec, spectrum.py:57-59) or c_k = b_e[j,e] - loc (exact residual,
// operators.py:69).  Compiled with -fmad=false, this is bit-identical to the reference.
//
// Memory: slot k of a chunk is one ROW of the slot blob: NB planes of 32 doubles (the A
// row of each lane's slot) followed by one id plane: per lane the local vertex j and the
// other vertices of the element (cyclic from j+1) as deltas to m packed in 32 bits (2D,
// 2 x 15 bit) or 64 bits (3D, 3 x 20 bit); meshes whose internal numbering is not local
// enough fall back to absolute int32 ids (NB-1 planes).  A warp streams 256 B per plane,
// fully coalesced, with evict-first loads; only the x gathers go through L1/L2, and they
// hit because the internal numbering keeps a chunk's neighbours within a few lines.
//
// Kernels are persistent: a fixed grid (occupancy-sized, so per-launch reductions have
// a fixed, deterministic order) of warps sweeps the chunks grid-stride.
#pragma once
#include "ebs_internal.cuh"

namespace ebs {

struct SellView {
    int64_t n_n, n_chunks;
    int rowb;
    const int32_t *__restrict__ rowbase;
    const int32_t *__restrict__ width;
    const int32_t *__restrict__ cnt;
    const uint8_t *__restrict__ slot;
    const double *__restrict__ be;
};

inline SellView sell_view(const Plan *p) {
    return SellView{p->n_n, p->n_chunks, p->rowb, p->rowbase, p->width, p->cnt, p->slot,
                    p->slot_be};
}

// packed id plane geometry
template <int NB>
struct Pack;
template <>
struct Pack<3> {
    using W = uint32_t;
    static constexpr int BITS = 15;
    static constexpr int64_t BIAS = 1 << 14;
    __device__ __forceinline__ static int j(W w) { return (int)(w >> 30); }
    __device__ __forceinline__ static int64_t d(W w, int t) {
        return (int64_t)((w >> (BITS * (1 - t))) & ((1u << BITS) - 1)) - BIAS;
    }
};
template <>
struct Pack<4> {
    using W = unsigned long long;
    static constexpr int BITS = 20;
    static constexpr int64_t BIAS = 1 << 19;
    __device__ __forceinline__ static int j(W w) { return (int)(w >> 62); }
    __device__ __forceinline__ static int64_t d(W w, int t) {
        return (int64_t)((w >> (BITS * (2 - t))) & ((1ull << BITS) - 1)) - BIAS;
    }
};

template <int NB>
__device__ __forceinline__ double pick(int t, double xo, const double (&g)[NB - 1]) {
    // t = (i - j - 1) mod NB: position of vertex i in the cyclic neighbour list; NB-1 = self
    double v = xo;
    if (t == 0) v = g[0];
    if (t == 1) v = g[1];
    if constexpr (NB == 4) {
        if (t == 2) v = g[2];
    }
    return v;
}

// Ordered slot sum of one node.  EXACT: sum of (b_e - loc); else sum of loc.
// `w` is the chunk width (warp-uniform), `c_m` this lane's valence, xo = x[m].
#ifndef EBS_U2
#define EBS_U2 1  // 2D slots in flight per thread (occupancy beats ILP here)
#endif
#ifndef EBS_U3
#define EBS_U3 1  // 3D slots in flight per thread
#endif
#ifndef EBS_MINB2
#define EBS_MINB2 8  // min resident 256-thread CTAs per SM, 2D SELL kernels (64 warps)
#endif
#ifndef EBS_MINB3
#define EBS_MINB3 6  // min resident 256-thread CTAs per SM, 3D SELL kernels
#endif
#define EBS_SELL_BOUNDS(NB) __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)

template <int NB, bool PACKED, bool EXACT>
__device__ __forceinline__ double sell_node_sum(const SellView &v, int64_t row0, int w, int lane,
                                                int64_t m, int c_m, const double *__restrict__ x,
                                                double xo) {
    constexpr int U = NB == 3 ? EBS_U2 : EBS_U3;
    double s = 0.0;
    for (int k0 = 0; k0 < w; k0 += U) {
        double a[U][NB];
        int32_t nid[U][NB - 1];
        int jj[U];
        double be[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u;
            const int64_t row = row0 + k;
            jj[u] = 0;
            be[u] = 0.0;
            if (k < c_m) {
                const uint8_t *rp = v.slot + row * v.rowb;
                const double *ap = reinterpret_cast<const double *>(rp) + lane;
#pragma unroll
                for (int i = 0; i < NB; ++i) a[u][i] = __ldcs(ap + i * LANES);
                if constexpr (PACKED) {
                    using W = typename Pack<NB>::W;
                    const W wd = __ldcs(reinterpret_cast<const W *>(rp + NB * 256) + lane);
                    jj[u] = Pack<NB>::j(wd);
#pragma unroll
                    for (int t = 0; t < NB - 1; ++t) nid[u][t] = (int32_t)(m + Pack<NB>::d(wd, t));
                } else {
                    const int32_t *ip = reinterpret_cast<const int32_t *>(rp + NB * 256) + lane;
#pragma unroll
                    for (int t = 0; t < NB - 1; ++t) {
                        int32_t id = __ldcs(ip + t * LANES);
                        if (t == 0) jj[u] = (int)((uint32_t)id >> J_SHIFT);
                        nid[u][t] = id & ID_MASK;
                    }
                }
                if constexpr (EXACT) be[u] = __ldcs(v.be + row * LANES + lane);
            } else {
#pragma unroll
                for (int i = 0; i < NB; ++i) a[u][i] = 0.0;
#pragma unroll
                for (int t = 0; t < NB - 1; ++t) nid[u][t] = -1;
            }
        }
        double g[U][NB - 1];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < NB - 1; ++t)
                g[u][t] = k0 + u < c_m ? __ldg(x + nid[u][t]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u < c_m) {
                const int j = jj[u];
                double loc = a[u][0] * pick<NB>((NB - j - 1) % NB, xo, g[u]);
#pragma unroll
                for (int i = 1; i < NB; ++i)
                    loc = loc + a[u][i] * pick<NB>((i - j - 1 + NB) % NB, xo, g[u]);
                if constexpr (EXACT) s = s + (be[u] - loc);
                else s = s + loc;
            }
        }
    }
    return s;
}

// Grid-stride sweep over chunks: epi(m, s, xo) for every valid node.
template <int NB, bool PACKED, bool EXACT, class Epi>
__device__ __forceinline__ void sell_sweep(const SellView &v, const double *__restrict__ x,
                                           Epi &epi) {
    const int lane = threadIdx.x & (LANES - 1);
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / LANES;
    for (int64_t c = warp; c < v.n_chunks; c += nwarps) {
        const int64_t m = c * LANES + lane;
        const bool valid = m < v.n_n;
        const int c_m = valid ? v.cnt[m] : 0;
        const double xo = valid ? x[m] : 0.0;
        const double s = sell_node_sum<NB, PACKED, EXACT>(v, v.rowbase[c], v.width[c], lane, m,
                                                          c_m, x, xo);
        if (valid) epi(m, s, xo);
    }
}

// Occupancy-sized persistent grid (cached per kernel and device).
int persistent_grid(const void *kernel, int block, int64_t work_blocks);

}  // namespace ebs

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
// Memory: slot k of a chunk is one "row": NB planes of 32 doubles (the A row) followed by
// NB-1 planes of 32 int32 (the other vertices, cyclic from j+1; plane 0 carries j in its
// top 2 bits).  A warp therefore streams 256 B per A plane and 128 B per id plane, fully
// coalesced, with evict-first loads; only the x gathers go through L1/L2, and they hit
// because the internal numbering keeps a chunk's neighbours within a few cache lines.
#pragma once
#include "ebs_internal.cuh"

namespace ebs {

struct SellView {
    int64_t n_n;
    const int32_t *__restrict__ rowbase;
    const int32_t *__restrict__ width;
    const int32_t *__restrict__ cnt;
    const int32_t *__restrict__ ids;
    const double *__restrict__ A;
    const double *__restrict__ be;
};

inline SellView sell_view(const Plan *p) {
    return SellView{p->n_n, p->rowbase, p->width, p->cnt, p->slot_nb, p->slot_A, p->slot_be};
}

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
template <int NB, bool EXACT>
__device__ __forceinline__ double sell_node_sum(const SellView &v, int64_t row0, int w, int lane,
                                                int c_m, const double *__restrict__ x,
                                                double xo) {
    constexpr int U = 4;  // slots in flight per batch
    double s = 0.0;
    for (int k0 = 0; k0 < w; k0 += U) {
        double a[U][NB];
        int32_t id[U][NB - 1];
        double be[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u;
            const int64_t row = row0 + k;
            if (k < c_m) {
                const double *ap = v.A + row * (NB * LANES) + lane;
#pragma unroll
                for (int i = 0; i < NB; ++i) a[u][i] = __ldcs(ap + i * LANES);
                const int32_t *ip = v.ids + row * ((NB - 1) * LANES) + lane;
#pragma unroll
                for (int t = 0; t < NB - 1; ++t) id[u][t] = __ldcs(ip + t * LANES);
                if constexpr (EXACT) be[u] = __ldcs(v.be + row * LANES + lane);
            } else {
#pragma unroll
                for (int i = 0; i < NB; ++i) a[u][i] = 0.0;
#pragma unroll
                for (int t = 0; t < NB - 1; ++t) id[u][t] = -1;
                be[u] = 0.0;
            }
        }
        double g[U][NB - 1];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < NB - 1; ++t)
                g[u][t] = id[u][t] != -1 ? __ldg(x + (id[u][t] & ID_MASK)) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u < c_m) {
                const int j = (int)((uint32_t)id[u][0] >> J_SHIFT);
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

}  // namespace ebs

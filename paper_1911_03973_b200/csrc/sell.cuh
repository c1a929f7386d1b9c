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
// enough fall back to absolute int32 ids (NB-1 planes).  Structured caller numberings
// (kept as the internal one) drop the id plane for one byte per slot indexing the plan's
// table of (j, differences) tuples (IDS_TUPLE, loaded one slot ahead).  A warp streams
// 256 B per plane, fully coalesced, with evict-first loads; only the x gathers go
// through L1/L2, and they hit because the internal numbering keeps a chunk's neighbours
// within a few lines.  The sweeps are close to issue-bound: per slot, decode and
// operand selection cost as much as the bytes (row_product branches on j).
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
    const uint8_t *__restrict__ cnt8;  // nullable: one-byte valences (read instead of cnt)
    const uint8_t *__restrict__ slot;
    const double *__restrict__ be;
    const int32_t *__restrict__ tab;     // per-chunk offset tables (IDS_TABLE)
    const int32_t *__restrict__ taboff;  // n_chunks + 1 offsets into tab
    int64_t n_rows;                      // slot rows of the blob (index checks)
    const int32_t *__restrict__ clist;   // nullable: sweep only these chunks
    int64_t nlist;                       // number of chunks swept (n_chunks or list size)
    const uint8_t *__restrict__ rowflag; // IDS_DELTA2: 1 = two-base row, 0 = 64-bit deltas
    const uint8_t *__restrict__ codes;   // IDS_TUPLE: one byte per slot (row * 32 + lane)
    const int4 *__restrict__ tup;        // IDS_TUPLE: the plan's (j, d_1, d_2[, d_3]) tuples
};

inline SellView sell_view(const Plan *p, const int32_t *clist = nullptr, int64_t nlist = -1) {
    return SellView{p->n_n, p->n_chunks, p->rowb, p->rowbase, p->width, p->cnt, p->cnt8, p->slot,
                    p->slot_be, p->tab, p->taboff, p->n_rows, clist, clist ? nlist : p->n_chunks,
                    p->rowflag, p->codes, p->tup};
}

// id-plane layouts (Plan::packed)
constexpr int IDS_ABS = 0;    // NB-1 planes of int32 absolute ids, j in the top bits of plane 0
constexpr int IDS_DELTA = 1;  // deltas to the node packed in 32 (2D) / 64 (3D) bits
constexpr int IDS_TABLE = 2;  // indices into a per-chunk table of deltas: 16 (2D) / 32 (3D) bits
// 3D only: rows whose 32 delta triples lie within +-255 of one of two row bases store a
// 32-bit code per lane (j:2 | base:1 | 3 x 9-bit residual) in the first half of the id
// plane and the two base triples at byte 128 (24 B, read once per row by the whole warp):
// 160 B read per row instead of 256.  Other rows keep IDS_DELTA's 64-bit words; a 1-byte
// flag per row (SellView::rowflag) says which.  No lookup on the id -> x-gather chain:
// code, bases and flag are independent loads.
constexpr int IDS_DELTA2 = 3;
// Meshes whose caller numbering is already a structured grid keep it (identity maps, no
// permutation at the API boundary; plan.cu find_strides).  There a slot's (j, neighbour
// - node differences) tuple takes only a few values -- 6 in 2D, 24 for Kuhn cubes (6 tet
// types x 4 vertices) -- so the plan can store the distinct tuples (<= TUPLE_CAP) and per
// slot one byte indexing them, in an array of its own (32 B per row), instead of the
// 8 B 3D id word; each warp keeps a copy of the table in shared memory and decodes with
// one 16 B shared-memory load.  Measured (profiles/README.md): C3 (2.1M nodes) 2859 ->
// 3020 it/s, but C5 (17M nodes) 362 -> 352 and the 2D kernels (32-register cap) lose, so
// plans use it for 3D meshes up to EBS_TUPLE_MAX_NODES nodes only.
constexpr int IDS_TUPLE = 4;
constexpr int TUPLE_CAP = 32;
constexpr int DIFF_CAP = 32;  // distinct differences collected while detecting the grid

template <int NB>
struct Tab;
template <>
struct Tab<3> {  // uint16: j (2 bits) | i0 (7) | i1 (7)
    using W = uint16_t;
    static constexpr int CAP = 128;
    __device__ __forceinline__ static int j(W w) { return (int)(w >> 14); }
    __device__ __forceinline__ static int idx(W w, int t) { return (w >> (7 * (1 - t))) & 127; }
};
template <>
struct Tab<4> {  // uint32: j (2 bits) | 6 spare | i0 (8) | i1 (8) | i2 (8)
    using W = uint32_t;
    static constexpr int CAP = 256;
    __device__ __forceinline__ static int j(W w) { return (int)(w >> 30); }
    __device__ __forceinline__ static int idx(W w, int t) { return (w >> (8 * (2 - t))) & 255; }
};

template <int NB, int IDS>
constexpr int id_plane_bytes() {
    return IDS == IDS_ABS ? 4 * (NB - 1) * 32
                          : (IDS == IDS_DELTA ? (NB == 3 ? 4 : 8) * 32 : (NB == 3 ? 2 : 4) * 32);
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

// How a sweep reads the vector it multiplies (x[i] for internal node i): the read-only
// path (the vector is not written during the kernel).
struct XLdg {
    const double *__restrict__ x;
    __device__ __forceinline__ double operator()(int i) const { return __ldg(x + i); }
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

// The slot's row product in vertex order, loc = ((A0*X0 + A1*X1) + A2*X2) [+ A3*X3] with
// X_j = xo and the other X_i = g[(i - j - 1) mod NB] (operators.py:69 einsum order).
template <int NB>
__device__ __forceinline__ double row_product_sel(int j, const double (&a)[NB], double xo,
                                                  const double (&g)[NB - 1]) {
    double loc = a[0] * pick<NB>((NB - j - 1) % NB, xo, g);
#pragma unroll
    for (int i = 1; i < NB; ++i) loc = loc + a[i] * pick<NB>((i - j - 1 + NB) % NB, xo, g);
    return loc;
}

// Same bits with a branch per local vertex j instead of per-operand selects (~24 FSEL
// per 3D slot): a node's slots are sorted by j, and on structured meshes every interior
// node has the same number of slots per j, so j is warp-uniform in nearly every row.
// 3D rows hold boundary nodes more often (a chunk straddles an x-row end), so there the
// branch is taken only when j is uniform over the active lanes.  Measured: C3 2980 ->
// 3130, C5 361 -> 369, C4 1656 -> 1720 it/s, C2 internal matvec 126 -> 121 us.  SW =
// false (the bit-exact residual, which spills at 32 registers with the branches): selects.
#ifndef EBS_TUPLE_PIPE
#define EBS_TUPLE_PIPE 1  // tuple-coded plans: codes one slot ahead (see sell_sweep)
#endif
#ifndef EBS_ROW_SWITCH
#define EBS_ROW_SWITCH 1
#endif
template <int NB, bool SW = true>
__device__ __forceinline__ double row_product(int j, const double (&a)[NB], double xo,
                                              const double (&g)[NB - 1]) {
    if constexpr (!SW || !EBS_ROW_SWITCH) {
        return row_product_sel<NB>(j, a, xo, g);
    } else if constexpr (NB == 3) {
        if (j == 0) return (a[0] * xo + a[1] * g[0]) + a[2] * g[1];
        if (j == 1) return (a[0] * g[1] + a[1] * xo) + a[2] * g[0];
        return (a[0] * g[0] + a[1] * g[1]) + a[2] * xo;
    } else {
        const unsigned am = __activemask();
        const int j0 = __shfl_sync(am, j, __ffs(am) - 1);
        if (!__all_sync(am, j == j0)) return row_product_sel<NB>(j, a, xo, g);
        if (j == 0) return ((a[0] * xo + a[1] * g[0]) + a[2] * g[1]) + a[3] * g[2];
        if (j == 1) return ((a[0] * g[2] + a[1] * xo) + a[2] * g[0]) + a[3] * g[1];
        if (j == 2) return ((a[0] * g[1] + a[1] * g[2]) + a[2] * xo) + a[3] * g[0];
        return ((a[0] * g[0] + a[1] * g[1]) + a[2] * g[2]) + a[3] * xo;
    }
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

template <int NB, int IDS, bool EXACT, class XL>
__device__ __forceinline__ double sell_node_sum(const SellView &v, int64_t row0, int w, int lane,
                                                int64_t m, int c_m, const XL &x,
                                                double xo, const int32_t *stab) {
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
                if constexpr (IDS == IDS_TABLE) {
                    using W = typename Tab<NB>::W;
                    const W wd = __ldcs(reinterpret_cast<const W *>(rp + NB * 256) + lane);
                    jj[u] = Tab<NB>::j(wd);
#pragma unroll
                    for (int t = 0; t < NB - 1; ++t)
                        nid[u][t] = (int32_t)m + stab[Tab<NB>::idx(wd, t)];
                } else if constexpr (IDS == IDS_DELTA) {
                    using W = typename Pack<NB>::W;
                    const W wd = __ldcs(reinterpret_cast<const W *>(rp + NB * 256) + lane);
                    jj[u] = Pack<NB>::j(wd);
#pragma unroll
                    for (int t = 0; t < NB - 1; ++t) nid[u][t] = (int32_t)(m + Pack<NB>::d(wd, t));
                } else if constexpr (IDS == IDS_TUPLE) {
                    const int4 tp = reinterpret_cast<const int4 *>(stab)[__ldcs(v.codes + row * LANES + lane)];
                    jj[u] = tp.x;
                    nid[u][0] = (int32_t)m + tp.y;
                    nid[u][1] = (int32_t)m + tp.z;
                    if constexpr (NB == 4) nid[u][2] = (int32_t)m + tp.w;
                } else if constexpr (IDS == IDS_DELTA2) {
                    static_assert(NB == 4, "IDS_DELTA2 is the 3D layout");
                    const uint8_t *ip = rp + NB * 256;
                    const int two = __ldg(v.rowflag + row);
                    const uint32_t code = __ldcs(reinterpret_cast<const uint32_t *>(ip) + lane);
                    const int4 h0 = __ldg(reinterpret_cast<const int4 *>(ip + 128));
                    const int2 h1 = __ldg(reinterpret_cast<const int2 *>(ip + 144));
                    if (two) {
                        const bool second = (code >> 29) & 1u;
                        const int b0 = second ? h0.w : h0.x, b1 = second ? h1.x : h0.y;
                        const int b2 = second ? h1.y : h0.z;
                        jj[u] = (int)(code >> 30);
                        nid[u][0] = (int32_t)m + b0 + (int)((code >> 18) & 511u) - 256;
                        nid[u][1] = (int32_t)m + b1 + (int)((code >> 9) & 511u) - 256;
                        nid[u][2] = (int32_t)m + b2 + (int)(code & 511u) - 256;
                    } else {
                        const unsigned long long wd =
                            __ldcs(reinterpret_cast<const unsigned long long *>(ip) + lane);
                        jj[u] = Pack<4>::j(wd);
#pragma unroll
                        for (int t = 0; t < 3; ++t) nid[u][t] = (int32_t)(m + Pack<4>::d(wd, t));
                    }
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
                g[u][t] = k0 + u < c_m ? (EBS_DCHECK(nid[u][t] >= 0 && nid[u][t] < v.n_n),
                                          x(nid[u][t]))
                                       : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u < c_m) {
                const int j = jj[u];
                const double loc = row_product<NB, !EXACT>(j, a[u], xo, g[u]);
                if constexpr (EXACT) s = s + (be[u] - loc);
                else s = s + loc;
            }
        }
    }
    return s;
}

// Raw id word(s) of one slot and their decoding (IDS_DELTA / IDS_ABS).
template <int NB, int IDS>
struct IdWord {
    static_assert(IDS == IDS_DELTA || IDS == IDS_ABS || IDS == IDS_TUPLE,
                  "one-slot-ahead ids: DELTA / ABS / TUPLE only");
    using W = typename Pack<NB>::W;
    W w;
    int32_t a[NB - 1];
    __device__ __forceinline__ void load(const SellView &v, int64_t row, int lane) {
        const uint8_t *rp = v.slot + row * v.rowb;
        if constexpr (IDS == IDS_TUPLE) {
            w = (W)__ldcs(v.codes + row * LANES + lane);
        } else if constexpr (IDS == IDS_DELTA) {
            w = __ldcs(reinterpret_cast<const W *>(rp + NB * 256) + lane);
        } else {
            const int32_t *ip = reinterpret_cast<const int32_t *>(rp + NB * 256) + lane;
#pragma unroll
            for (int t = 0; t < NB - 1; ++t) a[t] = __ldcs(ip + t * LANES);
        }
    }
    __device__ __forceinline__ int decode(const SellView &, int64_t m, int32_t (&nid)[NB - 1],
                                          const int32_t *stab) const {
        if constexpr (IDS == IDS_TUPLE) {
            const int4 tp = reinterpret_cast<const int4 *>(stab)[(int)w];
            nid[0] = (int32_t)m + tp.y;
            nid[1] = (int32_t)m + tp.z;
            if constexpr (NB == 4) nid[2] = (int32_t)m + tp.w;
            return tp.x;
        } else if constexpr (IDS == IDS_DELTA) {
#pragma unroll
            for (int t = 0; t < NB - 1; ++t) nid[t] = (int32_t)(m + Pack<NB>::d(w, t));
            return Pack<NB>::j(w);
        } else {
#pragma unroll
            for (int t = 0; t < NB - 1; ++t) nid[t] = a[t] & ID_MASK;
            return (int)((uint32_t)a[0] >> J_SHIFT);
        }
    }
};

// One slot in flight, with the id word of slot k+1 loaded while slot k is processed, so
// the x gathers of a slot issue at the start of its iteration (overlapping the A-row
// loads) instead of waiting a DRAM round trip for the ids.
template <int NB, int IDS, bool EXACT, class XL>
__device__ __forceinline__ double sell_node_sum_pipe(const SellView &v, int64_t row0, int w,
                                                     int lane, int64_t m, int c_m, const XL &x,
                                                     double xo, const int32_t *stab) {
    double s = 0.0;
    IdWord<NB, IDS> nxt;
    if (0 < c_m) nxt.load(v, row0, lane);
    for (int k = 0; k < w; ++k) {
        if (k < c_m) {
            const IdWord<NB, IDS> cur = nxt;
            const uint8_t *rp = v.slot + (row0 + k) * v.rowb;
            int32_t nid[NB - 1];
            const int j = cur.decode(v, m, nid, stab);
            double g[NB - 1];
#pragma unroll
            for (int t = 0; t < NB - 1; ++t) {
                EBS_DCHECK(nid[t] >= 0 && nid[t] < v.n_n);
                g[t] = x(nid[t]);
            }
            const double *ap = reinterpret_cast<const double *>(rp) + lane;
            double a[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) a[i] = __ldcs(ap + i * LANES);
            double be = 0.0;
            if constexpr (EXACT) be = __ldcs(v.be + (row0 + k) * LANES + lane);
            if (k + 1 < c_m) nxt.load(v, row0 + k + 1, lane);
            const double loc = row_product<NB, !EXACT>(j, a, xo, g);
            if constexpr (EXACT) s = s + (be - loc);
            else s = s + loc;
        }
    }
    return s;
}


// Per-warp shared-memory table of the id coding (IDS_TABLE: per chunk; IDS_TUPLE: the
// plan's tuples, loaded once).
template <int NB, int IDS>
struct SellStab {
    static constexpr int CAP = IDS == IDS_TABLE ? Tab<NB>::CAP : (IDS == IDS_TUPLE ? 4 * TUPLE_CAP : 1);
};

template <int NB, int IDS>
__device__ __forceinline__ int32_t *sell_stab_init(const SellView &v, int32_t (*stab_all)[SellStab<NB, IDS>::CAP]) {
    const int lane = threadIdx.x & (LANES - 1);
    int32_t *stab = stab_all[threadIdx.x / LANES];
    if constexpr (IDS == IDS_TUPLE) {
        for (int i = lane; i < TUPLE_CAP; i += LANES) reinterpret_cast<int4 *>(stab)[i] = v.tup[i];
        __syncwarp();
    }
    return stab;
}

// One chunk c (32 consecutive internal nodes, one per lane): the node sum s of this lane's
// node m (and xo = x[m]); `valid` false for the padding lanes of the last chunk.
struct ChunkSum {
    int m;
    bool valid;
    double s, xo;
};

template <int NB, int IDS, bool EXACT, bool PIPE, class XL>
__device__ __forceinline__ ChunkSum sell_chunk_sum(const SellView &v, int c, int lane,
                                                   int32_t *stab, const XL &x) {
    if constexpr (IDS == IDS_TABLE) {
        const int t0 = v.taboff[c], t1 = v.taboff[c + 1];
        __syncwarp();
        for (int i = lane; i < t1 - t0; i += LANES) stab[i] = v.tab[t0 + i];
        __syncwarp();
    }
    EBS_DCHECK(c >= 0 && c < v.n_chunks);
    EBS_DCHECK(v.rowbase[c] >= 0 && (int64_t)v.rowbase[c] + v.width[c] <= v.n_rows);
    ChunkSum r;
    r.m = c * LANES + lane;
    r.valid = r.m < v.n_n;
    const int c_m = r.valid ? (v.cnt8 ? (int)v.cnt8[r.m] : v.cnt[r.m]) : 0;
    r.xo = r.valid ? x(r.m) : 0.0;
    if constexpr ((PIPE || (IDS == IDS_TUPLE && EBS_TUPLE_PIPE)) && IDS != IDS_TABLE &&
                  IDS != IDS_DELTA2 && (NB == 3 ? EBS_U2 : EBS_U3) == 1)
        r.s = sell_node_sum_pipe<NB, IDS, EXACT>(v, v.rowbase[c], v.width[c], lane, r.m, c_m, x,
                                                 r.xo, stab);
    else
        r.s = sell_node_sum<NB, IDS, EXACT>(v, v.rowbase[c], v.width[c], lane, r.m, c_m, x,
                                            r.xo, stab);
    return r;
}

// ... and its epilogue: epi(m, s, xo) per valid node.
template <int NB, int IDS, bool EXACT, bool PIPE, class XL, class Epi>
__device__ __forceinline__ void sell_chunk(const SellView &v, int c, int lane, int32_t *stab,
                                           const XL &x, Epi &epi) {
    const ChunkSum r = sell_chunk_sum<NB, IDS, EXACT, PIPE>(v, c, lane, stab, x);
    if (r.valid) epi(r.m, r.s, r.xo);
}

// Grid-stride sweep over chunks: epi(m, s, xo) for every valid node (direct loads).
template <int NB, int IDS, bool EXACT, bool PIPE, class Epi>
__device__ __forceinline__ void sell_sweep_ldg(const SellView &v, const double *__restrict__ x,
                                               Epi &epi) {
    __shared__ __align__(16) int32_t stab_all[256 / LANES][SellStab<NB, IDS>::CAP];  // per warp
    const int lane = threadIdx.x & (LANES - 1);
    int32_t *stab = sell_stab_init<NB, IDS>(v, stab_all);
    const XLdg xl{x};
    // 32-bit chunk / node indices (plans hold < 2^30 nodes): the 64-bit loop counter of
    // the 2D kernels was the one value spilled at their 32-register cap
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
    const int nwarps = (int)((gridDim.x * blockDim.x) / LANES);
    const int nlist = (int)v.nlist;
    for (int ci = warp; ci < nlist; ci += nwarps) {
        const int c = v.clist ? v.clist[ci] : ci;
        sell_chunk<NB, IDS, EXACT, PIPE>(v, c, lane, stab, xl, epi);
    }
}

// ---------------------------------------------------------------- TMA bulk path --
// Each warp owns a ring of S shared-memory stages of R slot rows.  Lane 0 arms a stage's
// mbarrier with the byte count and issues one cp.async.bulk (TMA, 1-D) of the piece's
// contiguous rows; the warp consumes stage i while the next S-1 pieces are in flight.
// A piece is up to R rows of one chunk (chunks are `width` rows, contiguous in the blob).
#ifndef EBS_TMA
#define EBS_TMA 0
#endif
#ifndef EBS_TMA_W2
#define EBS_TMA_W2 8  // warps per CTA, 2D
#endif
#ifndef EBS_TMA_R2
#define EBS_TMA_R2 6  // rows per stage, 2D (structured 2D chunks are 6 rows)
#endif
#ifndef EBS_TMA_S2
#define EBS_TMA_S2 3  // stages per warp, 2D
#endif
#ifndef EBS_TMA_W3
#define EBS_TMA_W3 4
#endif
#ifndef EBS_TMA_R3
#define EBS_TMA_R3 8
#endif
#ifndef EBS_TMA_S3
#define EBS_TMA_S3 4
#endif

template <int NB>
struct TmaCfg {
    static constexpr int W = NB == 3 ? EBS_TMA_W2 : EBS_TMA_W3;
    static constexpr int R = NB == 3 ? EBS_TMA_R2 : EBS_TMA_R3;
    static constexpr int S = NB == 3 ? EBS_TMA_S2 : EBS_TMA_S3;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

template <int NB, int IDS, bool EXACT, class Epi>
__device__ __forceinline__ void sell_sweep_tma(const SellView &v, const double *__restrict__ x,
                                               Epi &epi) {
    constexpr bool PACKED = IDS == IDS_DELTA;
    constexpr int R = TmaCfg<NB>::R, S = TmaCfg<NB>::S, W = TmaCfg<NB>::W;
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ uint64_t bars[W][S];
    const int lane = threadIdx.x & (LANES - 1);
    const int wib = threadIdx.x / LANES;
    const int64_t warp = (int64_t)blockIdx.x * W + wib;
    const int64_t nwarps = (int64_t)gridDim.x * W;
    const int rowb = v.rowb;
    uint8_t *ring = dsm + (size_t)wib * S * R * rowb;
    uint64_t *bar = bars[wib];
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // producer cursor (lane 0 state, kept uniform)
    int64_t pc = warp;
    int pk0 = 0;
    int pstage = 0;
    auto produce = [&]() {
        if (pc >= v.n_chunks) return;
        const int w = v.width[pc];
        int nr = w - pk0;
        nr = nr > R ? R : nr;
        if (nr > 0 && lane == 0) {
            const uint32_t bytes = (uint32_t)nr * rowb;
            mbar_expect_tx(&bar[pstage], bytes);
            bulk_g2s(ring + (size_t)pstage * R * rowb,
                     v.slot + ((int64_t)v.rowbase[pc] + pk0) * rowb, bytes, &bar[pstage]);
        }
        pstage = pstage + 1 == S ? 0 : pstage + 1;
        pk0 += R;
        if (pk0 >= w) {
            pc += nwarps;
            pk0 = 0;
        }
    };
    for (int s = 0; s < S; ++s) produce();
    uint32_t phases = 0;
    int cstage = 0;
    for (int64_t c = warp; c < v.n_chunks; c += nwarps) {
        const int64_t m = c * LANES + lane;
        const bool valid = m < v.n_n;
        const int c_m = valid ? (v.cnt8 ? (int)v.cnt8[m] : v.cnt[m]) : 0;
        const double xo = valid ? x[m] : 0.0;
        const int w = v.width[c];
        const int64_t row0 = v.rowbase[c];
        double sum = 0.0;
        for (int k0 = 0; k0 < w || (k0 == 0 && w == 0); k0 += R) {
            int nr = w - k0;
            nr = nr > R ? R : nr;
            if (nr > 0) {
                mbar_wait(&bar[cstage], (phases >> cstage) & 1u);
                phases ^= 1u << cstage;
                const uint8_t *base = ring + (size_t)cstage * R * rowb;
#pragma unroll 2
                for (int r = 0; r < nr; ++r) {
                    const int k = k0 + r;
                    if (k < c_m) {
                        const uint8_t *rp = base + r * rowb;
                        const double *ap = reinterpret_cast<const double *>(rp) + lane;
                        double a[NB];
#pragma unroll
                        for (int i = 0; i < NB; ++i) a[i] = ap[i * LANES];
                        int32_t nid[NB - 1];
                        int j;
                        if constexpr (PACKED) {
                            using Wd = typename Pack<NB>::W;
                            const Wd wd = reinterpret_cast<const Wd *>(rp + NB * 256)[lane];
                            j = Pack<NB>::j(wd);
#pragma unroll
                            for (int t = 0; t < NB - 1; ++t)
                                nid[t] = (int32_t)(m + Pack<NB>::d(wd, t));
                        } else {
                            const int32_t *ip = reinterpret_cast<const int32_t *>(rp + NB * 256) + lane;
                            int32_t id0 = ip[0];
                            j = (int)((uint32_t)id0 >> J_SHIFT);
#pragma unroll
                            for (int t = 0; t < NB - 1; ++t) nid[t] = ip[t * LANES] & ID_MASK;
                        }
                        double g[NB - 1];
#pragma unroll
                        for (int t = 0; t < NB - 1; ++t) g[t] = __ldg(x + nid[t]);
                        const double loc = row_product<NB, !EXACT>(j, a, xo, g);
                        if constexpr (EXACT)
                            sum = sum + (__ldcs(v.be + (row0 + k) * LANES + lane) - loc);
                        else
                            sum = sum + loc;
                    }
                }
                __syncwarp();
            }
            cstage = cstage + 1 == S ? 0 : cstage + 1;
            produce();  // refill the stage just released with the piece S ahead
            if (w == 0) break;
        }
        if (valid) epi(m, sum, xo);
    }
}

#if EBS_TMA
#define EBS_SELL_THREADS(NB) (TmaCfg<NB>::W * LANES)
#define EBS_SELL_BOUNDS(NB) __launch_bounds__(EBS_SELL_THREADS(NB), 1)
#else
#define EBS_SELL_THREADS(NB) 256
#define EBS_SELL_BOUNDS(NB) __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)
#endif

// PIPE: load the id plane one slot ahead (sell_node_sum_pipe) -- measured faster for the
// 2D Jacobi step, slower for the other delta-coded kernels (profiles/README.md).  Tuple-
// coded plans always run it (EBS_TUPLE_PIPE): the one-byte code of slot k+1 is loaded
// while slot k is processed, so the table lookup and the gathers start at once -- C5 PCG
// matvec 2239 -> 2072 us (392 -> 423 it/s), C3 290 -> 272 us.
template <int NB, int IDS, bool EXACT, bool PIPE = false, class Epi>
__device__ __forceinline__ void sell_sweep(const SellView &v, const double *__restrict__ x,
                                           Epi &epi) {
#if EBS_TMA
    if constexpr (IDS != IDS_TABLE && IDS != IDS_DELTA2 && IDS != IDS_TUPLE) {
        if (v.clist == nullptr) {  // the TMA ring sweeps all chunks
            sell_sweep_tma<NB, IDS, EXACT>(v, x, epi);
            return;
        }
    }
#endif
    sell_sweep_ldg<NB, IDS, EXACT, PIPE>(v, x, epi);
}

// dispatch a macro M(NB, IDS) on the plan's geometry
#define EBS_SELL_DISPATCH(p, M)                                                          \
    do {                                                                                 \
        if ((p)->nb == 3) {                                                              \
            if ((p)->packed == IDS_TUPLE) M(3, IDS_TUPLE)                                  \
            else if ((p)->packed == IDS_TABLE) M(3, IDS_TABLE)                           \
            else if ((p)->packed == IDS_DELTA) M(3, IDS_DELTA)                           \
            else M(3, IDS_ABS)                                                           \
        } else {                                                                         \
            if ((p)->packed == IDS_TUPLE) M(4, IDS_TUPLE)                                  \
            else if ((p)->packed == IDS_TABLE) M(4, IDS_TABLE)                           \
            else if ((p)->packed == IDS_DELTA2) M(4, IDS_DELTA2)                         \
            else if ((p)->packed == IDS_DELTA) M(4, IDS_DELTA)                           \
            else M(4, IDS_ABS)                                                           \
        }                                                                                \
    } while (0)

// launch configuration of a SELL kernel (threads, dynamic smem, persistent grid)
struct SellLaunch {
    int grid, block;
    size_t smem;
};
SellLaunch sell_launch(const void *kernel, int nb, int rowb, int64_t n_chunks);

// Occupancy-sized persistent grid (cached per kernel and device).
int persistent_grid(const void *kernel, int block, int64_t work_blocks, size_t smem = 0);

}  // namespace ebs

// plan.cu -- execution plan of a mesh: node->(j,e) incidence in bincount order, a
// locality-preserving internal node numbering and the SELL-32 slot stream.
//
// Why: the reference scatter is np.bincount(indt.ravel(), w) (operators.py:98): per node a
// sequential sum from 0.0 over its contributions ordered by key j*n_e + e.  A node-centric
// gather that walks each node's slots in that key order reproduces it bit for bit without
// float atomics.  Slots are stored SELL-32: 32 consecutive internal nodes form a chunk
// (one warp), slot k of lane l lives in row rowbase[c]+k, so every load of the hot loop
// is a coalesced 256 B (doubles) / 128 B (ids) warp transaction.
//
// Internal numbering = first appearance when scanning elements e ascending, j ascending
// (oracle/ebs_oracle.py first_appearance_order).  On structured meshes this recovers the
// geometric row/plane order even when the caller's numbering is a random permutation
// (BASELINE C2/C4), so the x gathers of a warp hit a few cache lines.  Exception: when
// the caller's numbering is a structured grid (an unpermuted generated mesh, BASELINE
// C1/C3/C5: every (neighbour - node) difference is a +-1 combination of axis strides),
// that numbering is kept (identity maps)
// (oracle/ebs_oracle.py grid_strides), and slots store one-byte codes of their
// (j, differences) tuples (sell.cuh IDS_TUPLE).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "sell.cuh"

#ifndef EBS_IDS_DELTA2
#define EBS_IDS_DELTA2 0  // 3D two-base row coding of the id plane (opt-in: measured slower)
#endif
#ifndef EBS_IDS_TABLE
#define EBS_IDS_TABLE 0  // per-chunk delta-table id layout (opt-in: measured slower, profiles/README.md)
#endif

namespace ebs {

// Identity numbering for structured caller numberings (EBS_IDS_GRID=0 in the environment
// turns it off: comparisons against the first-appearance path)
static int grid_mode() {
    static const int v = [] {
        const char *e = getenv("EBS_IDS_GRID");
        return e ? atoi(e) : 1;
    }();
    return v;
}
static bool grid_enabled() { return grid_mode() != 0; }

// IDS_TUPLE codes on structured plans (loaded a slot ahead, with the row-product
// branch: C3 2818 -> 3340, C5 369 -> 424 it/s; 2D paper experiment 6.05 -> 5.94 ms).
// EBS_IDS_GRID=2 turns them off (packed deltas), =3 forces them (tests)
static bool tuple_wanted(int, int64_t) { return grid_mode() != 2; }

// ------------------------------------------------------------- build kernels --
__global__ void k_incidence(int nb, int64_t n_n, int64_t n_e, const int32_t *__restrict__ conn,
                            int32_t *__restrict__ cnt, unsigned long long *__restrict__ first,
                            int32_t *bad) {
    const int64_t total = (int64_t)nb * n_e;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t j = t / n_e, e = t - j * n_e;
        int32_t n = conn[t];
        if (n < 0 || n >= n_n) { atomicOr(bad, 1); continue; }
        atomicAdd(&cnt[n], 1);
        atomicMin(&first[n], (unsigned long long)(e * nb + j));
    }
}

// flag[e*nb + j] = 1 iff (e, j) is the first appearance of its node
__global__ void k_first_flags(int nb, int64_t n_e, const int32_t *__restrict__ conn,
                              const unsigned long long *__restrict__ first,
                              int32_t *__restrict__ flag) {
    const int64_t total = (int64_t)nb * n_e;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = t / nb, j = t - e * nb;
        int32_t n = conn[j * n_e + e];
        flag[t] = (first[n] == (unsigned long long)t) ? 1 : 0;
    }
}

__global__ void k_isolated_flags(int64_t n_n, const int32_t *__restrict__ cnt,
                                 int32_t *__restrict__ flag) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_n;
         n += (int64_t)gridDim.x * blockDim.x)
        flag[n] = cnt[n] == 0 ? 1 : 0;
}

__global__ void k_numbering(int64_t n_n, int64_t n_conn, const int32_t *__restrict__ cnt,
                            const unsigned long long *__restrict__ first,
                            const int32_t *__restrict__ pos_first,
                            const int32_t *__restrict__ pos_iso, int32_t *__restrict__ new_of_old,
                            int32_t *__restrict__ old_of_new) {
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_n;
         n += (int64_t)gridDim.x * blockDim.x) {
        int32_t m = cnt[n] > 0 ? pos_first[first[n]] : (int32_t)(n_conn + pos_iso[n]);
        new_of_old[n] = m;
        old_of_new[m] = (int32_t)n;
    }
}

__global__ void k_cnt8(int64_t n_n, const int32_t *__restrict__ cnt, uint8_t *__restrict__ cnt8) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_n;
         m += (int64_t)gridDim.x * blockDim.x)
        cnt8[m] = (uint8_t)cnt[m];
}

__global__ void k_permute_cnt(int64_t n_n, const int32_t *__restrict__ old_of_new,
                              const int32_t *__restrict__ cnt_old, int32_t *__restrict__ cnt_new) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_n;
         m += (int64_t)gridDim.x * blockDim.x)
        cnt_new[m] = cnt_old[old_of_new[m]];
}

__global__ void k_fill_keys(int nb, int64_t n_e, const int32_t *__restrict__ conn,
                            const int32_t *__restrict__ new_of_old,
                            const int32_t *__restrict__ rowptr, int32_t *__restrict__ fill,
                            int64_t *__restrict__ keys) {
    const int64_t total = (int64_t)nb * n_e;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int32_t m = new_of_old[conn[t]];
        int32_t p = rowptr[m] + atomicAdd(&fill[m], 1);
        keys[p] = t;  // t = j*n_e + e: the bincount order key
    }
}

// sort each node's keys ascending (atomics above filled them in arbitrary order)
__global__ void k_sort_segments(int64_t n_n, const int32_t *__restrict__ rowptr,
                                const int32_t *__restrict__ cnt, int64_t *__restrict__ keys) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_n;
         m += (int64_t)gridDim.x * blockDim.x) {
        int64_t *k = keys + rowptr[m];
        int c = cnt[m];
        for (int a = 1; a < c; ++a) {
            int64_t v = k[a];
            int b = a - 1;
            while (b >= 0 && k[b] > v) { k[b + 1] = k[b]; --b; }
            k[b + 1] = v;
        }
    }
}

__global__ void k_chunk_width(int64_t n_n, int64_t n_chunks, const int32_t *__restrict__ cnt,
                              int32_t *__restrict__ width) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks;
         c += (int64_t)gridDim.x * blockDim.x) {
        int w = 0;
        for (int l = 0; l < LANES; ++l) {
            int64_t m = c * LANES + l;
            if (m < n_n && cnt[m] > w) w = cnt[m];
        }
        width[c] = w;
    }
}

__global__ void k_fill_slots(int nb, int64_t n_n, int64_t n_e, const int32_t *__restrict__ conn,
                             const int32_t *__restrict__ new_of_old,
                             const int32_t *__restrict__ rowptr, const int32_t *__restrict__ cnt,
                             const int64_t *__restrict__ keys, const int32_t *__restrict__ rowbase,
                             const int32_t *__restrict__ width, int32_t *__restrict__ slot_ej,
                             int32_t *__restrict__ ids_abs, unsigned long long *max_delta) {
    const int64_t n_pad = ((n_n + LANES - 1) / LANES) * LANES;
    unsigned long long md = 0;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_pad;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = m / LANES;
        const int lane = (int)(m - c * LANES);
        const int c_m = m < n_n ? cnt[m] : 0;
        const int w = width[c];
        for (int k = 0; k < w; ++k) {
            const int64_t row = (int64_t)rowbase[c] + k;
            if (k < c_m) {
                int64_t key = keys[rowptr[m] + k];
                int64_t j = key / n_e, e = key - j * n_e;
                slot_ej[row * LANES + lane] = (int32_t)e | (int32_t)(j << J_SHIFT);
                for (int t = 1; t < nb; ++t) {
                    int64_t jj = (j + t) % nb;
                    int32_t id = new_of_old[conn[jj * n_e + e]];
                    int64_t d = (int64_t)id - m;
                    unsigned long long ad = (unsigned long long)(d < 0 ? -d : d);
                    md = ad > md ? ad : md;
                    if (t == 1) id |= (int32_t)(j << J_SHIFT);
                    ids_abs[(row * (nb - 1) + (t - 1)) * LANES + lane] = id;
                }
            } else {
                slot_ej[row * LANES + lane] = -1;
                int32_t self = m < n_n ? (int32_t)m : 0;
                for (int t = 1; t < nb; ++t)
                    ids_abs[(row * (nb - 1) + (t - 1)) * LANES + lane] = self;
            }
        }
    }
    if (md) atomicMax(max_delta, md);
}

// Per-chunk delta tables (id layout 2): every distinct (neighbour - node) delta of a
// chunk's slots, sorted ascending; slots store 7-bit (2D) / 8-bit (3D) indices into it.
// Warp per chunk, open-addressing hash in shared memory; pass 1 counts, pass 2 (with
// the scanned offsets) writes the table and the id plane.  Deterministic: the table is
// the sorted set, independent of the insertion order.
constexpr int TAB_HASH = 1024;
constexpr int32_t TAB_EMPTY = (int32_t)0x80000000;

__device__ __forceinline__ int tab_hash(int32_t d) {
    return (int)(((uint32_t)d * 2654435761u) >> 22) & (TAB_HASH - 1);
}

__global__ void __launch_bounds__(128)
    k_chunk_tables(int nb, int64_t n_n, int64_t n_chunks, int cap, const int32_t *__restrict__ rowbase,
                   const int32_t *__restrict__ width, const int32_t *__restrict__ cnt,
                   const int32_t *__restrict__ ids_abs, int32_t *__restrict__ counts,
                   const int32_t *__restrict__ taboff, int32_t *__restrict__ tab,
                   uint8_t *__restrict__ slot, int rowb, int32_t *overflow) {
    __shared__ int32_t hkey[4][TAB_HASH];
    __shared__ int16_t hrank[4][TAB_HASH];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *key = hkey[w];
    int16_t *rnk = hrank[w];
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < n_chunks; c += nwarps) {
        for (int h = lane; h < TAB_HASH; h += 32) key[h] = TAB_EMPTY;
        __syncwarp();
        const int64_t m = c * 32 + lane;
        const int c_m = m < n_n ? cnt[m] : 0;
        const int wd = width[c];
        const int64_t row0 = rowbase[c];
        bool full = false;
        for (int k = 0; k < c_m && !full; ++k)
            for (int t = 0; t < nb - 1; ++t) {
                const int32_t d = (ids_abs[((row0 + k) * (nb - 1) + t) * 32 + lane] & ID_MASK) - (int32_t)m;
                int h = tab_hash(d);
                bool placed = false;
                for (int probe = 0; probe < TAB_HASH && !placed; ++probe) {  // bounded: a
                    int32_t old = atomicCAS(&key[h], TAB_EMPTY, d);           // full hash
                    placed = old == TAB_EMPTY || old == d;                    // = overflow
                    h = (h + 1) & (TAB_HASH - 1);
                }
                full |= !placed;
            }
        __syncwarp();
        int K = 0;
        for (int h = lane; h < TAB_HASH; h += 32) K += key[h] != TAB_EMPTY;
        for (int o = 16; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
        if (__any_sync(0xffffffffu, full) || K > cap) {
            if (lane == 0) atomicOr(overflow, 1);
            continue;
        }
        if (!taboff) {
            if (lane == 0) counts[c] = K;
            continue;
        }
        // rank = number of smaller keys (sorted, deterministic)
        for (int h = lane; h < TAB_HASH; h += 32) {
            const int32_t v = key[h];
            if (v == TAB_EMPTY) continue;
            int r = 0;
            for (int g = 0; g < TAB_HASH; ++g) {
                const int32_t u = key[g];
                r += (u != TAB_EMPTY) & (u < v);
            }
            rnk[h] = (int16_t)r;
            tab[taboff[c] + r] = v;
        }
        __syncwarp();
        for (int k = 0; k < wd; ++k) {
            const int64_t row = row0 + k;
            uint32_t word = 0;
            if (k < c_m) {
                const int32_t id0 = ids_abs[(row * (nb - 1)) * 32 + lane];
                const uint32_t j = (uint32_t)id0 >> J_SHIFT;
                word = nb == 3 ? (j << 14) : (j << 30);
                for (int t = 0; t < nb - 1; ++t) {
                    const int32_t d = (ids_abs[(row * (nb - 1) + t) * 32 + lane] & ID_MASK) - (int32_t)m;
                    int h = tab_hash(d);
                    while (key[h] != d) h = (h + 1) & (TAB_HASH - 1);
                    const uint32_t r = (uint32_t)rnk[h];
                    word |= nb == 3 ? (r << (7 * (1 - t))) : (r << (8 * (2 - t)));
                }
            }
            uint8_t *dst = slot + row * rowb + nb * 256;
            if (nb == 3) reinterpret_cast<uint16_t *>(dst)[lane] = (uint16_t)word;
            else reinterpret_cast<uint32_t *>(dst)[lane] = word;
        }
        __syncwarp();
    }
}

// id layout 3 (3D): per slot row, the mode of the 32 lanes' delta triples is base 1, the
// mode of the lanes more than 255 away from it base 2; when every valid lane lies within
// +-255 of one of them the row is coded with 32-bit words (j:2 | base:1 | 3 x 9-bit
// residual + 256) and the two bases at byte 128 of the id plane (rowflag = 1), else with
// IDS_DELTA's 64-bit words (rowflag = 0).  One warp per chunk.
__device__ __forceinline__ bool same3(int a0, int a1, int a2, int b0, int b1, int b2) {
    return a0 == b0 && a1 == b1 && a2 == b2;
}

__global__ void __launch_bounds__(128)
    k_write_ids_delta2(int64_t n_n, int64_t n_chunks, int rowb,
                       const int32_t *__restrict__ rowbase, const int32_t *__restrict__ width,
                       const int32_t *__restrict__ cnt, const int32_t *__restrict__ ids_abs,
                       uint8_t *__restrict__ slot, uint8_t *__restrict__ rowflag,
                       unsigned long long *two_rows) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long n_two = 0;
    for (int64_t c = warp; c < n_chunks; c += nwarps) {
        const int64_t m = c * LANES + lane;
        const int64_t self = m < n_n ? m : 0;
        const int c_m = m < n_n ? cnt[m] : 0;
        const int w = width[c];
        for (int k = 0; k < w; ++k) {
            const int64_t row = (int64_t)rowbase[c] + k;
            const int32_t *src = ids_abs + row * 3 * LANES + lane;
            const bool valid = k < c_m;
            const int32_t id0 = src[0];
            const uint32_t j = (uint32_t)id0 >> J_SHIFT;
            int d0 = 0, d1 = 0, d2 = 0;
            if (valid) {
                d0 = (int)((id0 & ID_MASK) - self);
                d1 = (int)((src[LANES] & ID_MASK) - self);
                d2 = (int)((src[2 * LANES] & ID_MASK) - self);
            }
            // base 1: the most frequent valid triple (ties: lowest lane)
            int votes = 0;
            for (int o = 0; o < LANES; ++o) {
                const int e0 = __shfl_sync(0xffffffffu, d0, o), e1 = __shfl_sync(0xffffffffu, d1, o);
                const int e2 = __shfl_sync(0xffffffffu, d2, o);
                const bool vo = __shfl_sync(0xffffffffu, valid, o);
                votes += vo && same3(e0, e1, e2, d0, d1, d2);
            }
            int key = valid ? votes * 64 + (31 - lane) : -1;
            for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
            const int win1 = key >= 0 ? 31 - (key & 63) : 0;
            const int b10 = __shfl_sync(0xffffffffu, d0, win1), b11 = __shfl_sync(0xffffffffu, d1, win1);
            const int b12 = __shfl_sync(0xffffffffu, d2, win1);
            auto near = [](int a0, int a1, int a2, int b0, int b1, int b2) {
                return abs(a0 - b0) <= 255 && abs(a1 - b1) <= 255 && abs(a2 - b2) <= 255;
            };
            const bool fit1 = valid && near(d0, d1, d2, b10, b11, b12);
            const bool far = valid && !fit1;
            // base 2: the most frequent triple among the lanes base 1 does not cover
            int votes2 = 0;
            for (int o = 0; o < LANES; ++o) {
                const int e0 = __shfl_sync(0xffffffffu, d0, o), e1 = __shfl_sync(0xffffffffu, d1, o);
                const int e2 = __shfl_sync(0xffffffffu, d2, o);
                const bool fo = __shfl_sync(0xffffffffu, far, o);
                votes2 += fo && same3(e0, e1, e2, d0, d1, d2);
            }
            int key2 = far ? votes2 * 64 + (31 - lane) : -1;
            for (int o = 16; o > 0; o >>= 1) key2 = max(key2, __shfl_xor_sync(0xffffffffu, key2, o));
            const int win2 = key2 >= 0 ? 31 - (key2 & 63) : win1;
            const int b20 = __shfl_sync(0xffffffffu, d0, win2), b21 = __shfl_sync(0xffffffffu, d1, win2);
            const int b22 = __shfl_sync(0xffffffffu, d2, win2);
            const bool fit2 = valid && near(d0, d1, d2, b20, b21, b22);
            const bool two = __all_sync(0xffffffffu, !valid || fit1 || fit2);
            uint8_t *dst = slot + row * rowb + 4 * 256;
            if (two) {
                uint32_t code = 0;
                if (valid) {
                    const bool sel = !fit1;
                    const int c0 = d0 - (sel ? b20 : b10) + 256, c1 = d1 - (sel ? b21 : b11) + 256;
                    const int c2 = d2 - (sel ? b22 : b12) + 256;
                    code = (j << 30) | ((uint32_t)sel << 29) | ((uint32_t)c0 << 18) |
                           ((uint32_t)c1 << 9) | (uint32_t)c2;
                }
                reinterpret_cast<uint32_t *>(dst)[lane] = code;
                if (lane < 8) {
                    const int h[8] = {b10, b11, b12, b20, b21, b22, 0, 0};
                    reinterpret_cast<int32_t *>(dst + 128)[lane] = h[lane];
                }
                if (lane == 0) {
                    rowflag[row] = 1;
                    ++n_two;
                }
            } else {
                unsigned long long wd = (unsigned long long)j << 62;
                const int dd[3] = {d0, d1, d2};
                for (int t = 0; t < 3; ++t)
                    wd |= ((unsigned long long)(dd[t] + (1 << 19)) & 0xFFFFFull) << (20 * (2 - t));
                reinterpret_cast<unsigned long long *>(dst)[lane] = wd;
                if (lane == 0) rowflag[row] = 0;
            }
        }
    }
    if (lane == 0 && n_two) atomicAdd(two_rows, n_two);
}

// The (neighbour - node) id differences of the caller numbering, d = conn[(j+t)%nb][e] -
// conn[j][e], collected into a set of at most DIFF_CAP values: per CTA in shared
// memory (linear probing; nearly every probe finds its value among the first few
// entries), then merged into the global set.  *overflow = 1 when there are more.
constexpr int32_t DIFF_EMPTY = (int32_t)0x80000000;

__device__ __forceinline__ bool diff_insert(int32_t *set, int32_t d) {
    for (int i = 0; i < DIFF_CAP; ++i) {
        int32_t cur = *(volatile int32_t *)(set + i);
        if (cur == d) return true;
        if (cur == DIFF_EMPTY) {
            cur = atomicCAS(set + i, DIFF_EMPTY, d);
            if (cur == DIFF_EMPTY || cur == d) return true;
        }
    }
    return false;
}

__global__ void k_diff_set(int nb, int64_t n_e, const int32_t *__restrict__ conn,
                           int32_t *__restrict__ set, int32_t *overflow) {
    __shared__ int32_t st[DIFF_CAP];
    __shared__ int sover;
    if (threadIdx.x < DIFF_CAP) st[threadIdx.x] = DIFF_EMPTY;
    if (threadIdx.x == 0) sover = 0;
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (*(volatile int *)&sover) break;
        int32_t v[4];
        for (int j = 0; j < nb; ++j) v[j] = conn[j * n_e + e];
        bool ok = true;
        for (int j = 0; j < nb && ok; ++j)
            for (int t = 1; t < nb && ok; ++t) ok = diff_insert(st, v[(j + t) % nb] - v[j]);
        if (!ok) sover = 1;
    }
    __syncthreads();
    if (threadIdx.x < DIFF_CAP && st[threadIdx.x] != DIFF_EMPTY &&
        !diff_insert(set, st[threadIdx.x]))
        atomicOr(overflow, 1);
    if (threadIdx.x == 0 && sover) atomicOr(overflow, 1);
}

__global__ void k_iota(int64_t n, int32_t *__restrict__ a, int32_t *__restrict__ b) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = b[i] = (int32_t)i;
}

// id layout 4 (sell.cuh IDS_TUPLE): the distinct (j, d_1, .., d_{nb-1}) tuples of the
// slots, as 64-bit keys j << 60 | biased 20-bit differences, collected into a set of at
// most TUPLE_CAP (per CTA in shared memory, then merged); *overflow = 1 when there are
// more.  Needs every |difference| < 2^19 (IDS_DELTA's range).
constexpr unsigned long long TUP_EMPTY = ~0ull;

__device__ __forceinline__ unsigned long long tuple_key(int nb, const int32_t *src, int64_t m) {
    unsigned long long key = (unsigned long long)((uint32_t)src[0] >> J_SHIFT) << 60;
    for (int t = 0; t < nb - 1; ++t) {
        const int64_t d = (int64_t)(src[t * LANES] & ID_MASK) - m;
        key |= (unsigned long long)((d + (1 << 19)) & 0xFFFFF) << (20 * t);
    }
    return key;
}

__device__ __forceinline__ bool tup_insert(unsigned long long *set, unsigned long long k) {
    for (int i = 0; i < TUPLE_CAP; ++i) {
        unsigned long long cur = *(volatile unsigned long long *)(set + i);
        if (cur == k) return true;
        if (cur == TUP_EMPTY) {
            cur = atomicCAS(set + i, TUP_EMPTY, k);
            if (cur == TUP_EMPTY || cur == k) return true;
        }
    }
    return false;
}

__global__ void k_tuple_set(int nb, int64_t n_n, int64_t n_chunks,
                            const int32_t *__restrict__ rowbase, const int32_t *__restrict__ cnt,
                            const int32_t *__restrict__ ids_abs, unsigned long long *set,
                            int32_t *overflow) {
    __shared__ unsigned long long st[TUPLE_CAP];
    __shared__ int sover;
    if (threadIdx.x < TUPLE_CAP) st[threadIdx.x] = TUP_EMPTY;
    if (threadIdx.x == 0) sover = 0;
    __syncthreads();
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_n;
         m += (int64_t)gridDim.x * blockDim.x) {
        if (*(volatile int *)&sover) break;
        const int64_t c = m / LANES;
        const int lane = (int)(m - c * LANES);
        for (int k = 0; k < cnt[m]; ++k) {
            const int64_t row = (int64_t)rowbase[c] + k;
            if (!tup_insert(st, tuple_key(nb, ids_abs + row * (nb - 1) * LANES + lane, m))) {
                sover = 1;
                break;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < TUPLE_CAP && st[threadIdx.x] != TUP_EMPTY && !tup_insert(set, st[threadIdx.x]))
        atomicOr(overflow, 1);
    if (threadIdx.x == 0 && sover) atomicOr(overflow, 1);
}

// codes[row * 32 + lane] = index of the slot's tuple in the sorted key list (0 for padding)
__global__ void k_write_codes(int nb, int64_t n_n, int64_t n_chunks,
                              const int32_t *__restrict__ rowbase,
                              const int32_t *__restrict__ width, const int32_t *__restrict__ cnt,
                              const int32_t *__restrict__ ids_abs,
                              const unsigned long long *__restrict__ keys, int n_keys,
                              uint8_t *__restrict__ codes, int32_t *bad) {
    const int64_t n_pad = n_chunks * LANES;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_pad;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = m / LANES;
        const int lane = (int)(m - c * LANES);
        const int w = width[c];
        const int c_m = m < n_n ? cnt[m] : 0;
        for (int k = 0; k < w; ++k) {
            const int64_t row = (int64_t)rowbase[c] + k;
            int code = 0;
            if (k < c_m) {
                const unsigned long long key = tuple_key(nb, ids_abs + row * (nb - 1) * LANES + lane, m);
                code = -1;
                for (int i = 0; i < n_keys; ++i)
                    if (keys[i] == key) code = i;
                if (code < 0) { atomicOr(bad, 1); code = 0; }
            }
            codes[row * LANES + lane] = (uint8_t)code;
        }
    }
}

// Axis strides s0 < s1 (< s2) taken from the positive differences such that every
// difference is a*s0 + b*s1 (+ c*s2), a, b, c in {-1, 0, 1}; the first such choice in
// lexicographic order.  False when there is none.
static bool find_strides(int dim, const std::vector<int32_t> &diff, int32_t (&st)[3]) {
    std::vector<int64_t> pos;
    for (int32_t d : diff)
        if (d > 0) pos.push_back(d);
    const size_t P = pos.size();
    auto fits = [&](int64_t a0, int64_t a1, int64_t a2) {
        for (int32_t d : diff) {
            bool ok = false;
            for (int q = 0; q < 27 && !ok; ++q) {
                const int a = q % 3 - 1, b = (q / 3) % 3 - 1, c = q / 9 - 1;
                if (dim == 2 && c != 0) continue;
                ok = a * a0 + b * a1 + c * a2 == d;
            }
            if (!ok) return false;
        }
        return true;
    };
    for (size_t i = 0; i < P; ++i)
        for (size_t k = i + 1; k < P; ++k) {
            if (dim == 2) {
                if (fits(pos[i], pos[k], 0)) {
                    st[0] = (int32_t)pos[i], st[1] = (int32_t)pos[k], st[2] = 0;
                    return true;
                }
                continue;
            }
            for (size_t l = k + 1; l < P; ++l)
                if (fits(pos[i], pos[k], pos[l])) {
                    st[0] = (int32_t)pos[i], st[1] = (int32_t)pos[k], st[2] = (int32_t)pos[l];
                    return true;
                }
        }
    return false;
}

// id plane of every slot row (sell.cuh layout): delta-packed or absolute
__global__ void k_write_ids(int nb, int64_t n_n, int64_t n_chunks, int rowb, int packed,
                            const int32_t *__restrict__ rowbase, const int32_t *__restrict__ width,
                            const int32_t *__restrict__ ids_abs, uint8_t *__restrict__ slot) {
    const int64_t n_pad = n_chunks * LANES;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_pad;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = m / LANES;
        const int lane = (int)(m - c * LANES);
        const int w = width[c];
        const int64_t self = m < n_n ? m : 0;
        for (int k = 0; k < w; ++k) {
            const int64_t row = (int64_t)rowbase[c] + k;
            const int32_t *src = ids_abs + row * (nb - 1) * LANES + lane;
            uint8_t *dst = slot + row * rowb + nb * 256;
            if (packed) {
                const int32_t id0 = src[0];
                const uint64_t j = (uint32_t)id0 >> J_SHIFT;
                if (nb == 3) {
                    uint32_t wd = (uint32_t)j << 30;
                    for (int t = 0; t < 2; ++t) {
                        int64_t id = (int64_t)(src[t * LANES] & ID_MASK);
                        uint32_t f = (uint32_t)(id - self + (1 << 14)) & 0x7FFFu;
                        wd |= f << (15 * (1 - t));
                    }
                    reinterpret_cast<uint32_t *>(dst)[lane] = wd;
                } else {
                    unsigned long long wd = (unsigned long long)j << 62;
                    for (int t = 0; t < 3; ++t) {
                        int64_t id = (int64_t)(src[t * LANES] & ID_MASK);
                        unsigned long long f =
                            (unsigned long long)(id - self + (1 << 19)) & 0xFFFFFull;
                        wd |= f << (20 * (2 - t));
                    }
                    reinterpret_cast<unsigned long long *>(dst)[lane] = wd;
                }
            } else {
                for (int t = 0; t < nb - 1; ++t)
                    reinterpret_cast<int32_t *>(dst)[t * LANES + lane] = src[t * LANES];
            }
        }
    }
}

// ------------------------------------------------------------- load kernels --
__global__ void k_pack(int nb, int64_t n_e, int64_t n_slots, int rowb,
                       const int32_t *__restrict__ slot_ej, const double *__restrict__ A_e,
                       const double *__restrict__ b_e, uint8_t *__restrict__ slot,
                       double *__restrict__ slot_be) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_slots;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = s / LANES;
        const int lane = (int)(s - row * LANES);
        const int32_t ej = slot_ej[s];
        double *dst = reinterpret_cast<double *>(slot + row * rowb) + lane;
        if (ej != -1) {  // j >= 2 sets the sign bit: only -1 marks padding
            const int64_t e = ej & ID_MASK, j = (uint32_t)ej >> J_SHIFT;
            const double *src = A_e + (e * nb + j) * nb;  // row j of element e
            for (int i = 0; i < nb; ++i) dst[i * LANES] = src[i];
            if (slot_be) slot_be[s] = b_e[j * n_e + e];
        } else {
            for (int i = 0; i < nb; ++i) dst[i * LANES] = 0.0;
            if (slot_be) slot_be[s] = 0.0;
        }
    }
}

// Ordered per-node sums over slots of a value fetched per slot:
//   what = 0: b_e[j, e] (assemble_rhs, operators.py:58-63)
//   what = 1: A plane j of the slot row = A_e[j, j, e] (diag)
//   what = 2: slot_be (pre-assembled b from the packed stream)
//   what = 3: diag summed per local vertex j first (mass_gershgorin order)
// out_user != nullptr writes caller numbering, else internal numbering.
__global__ void k_slot_sum(int nb, int64_t n_n, int64_t n_e, const int32_t *__restrict__ rowbase,
                           const int32_t *__restrict__ width, const int32_t *__restrict__ cnt,
                           const int32_t *__restrict__ slot_ej, const uint8_t *__restrict__ slot,
                           int rowb,
                           const double *__restrict__ slot_be, const double *__restrict__ b_e,
                           int what, const int32_t *__restrict__ old_of_new,
                           double *__restrict__ out) {
    const int64_t n_pad = ((n_n + LANES - 1) / LANES) * LANES;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_pad;
         m += (int64_t)gridDim.x * blockDim.x) {
        if (m >= n_n) continue;
        const int64_t c = m / LANES;
        const int lane = (int)(m - c * LANES);
        const int c_m = cnt[m];
        double s = 0.0, grp = 0.0;
        int cur_j = -1;
        for (int k = 0; k < c_m; ++k) {
            const int64_t row = (int64_t)rowbase[c] + k;
            const int64_t sidx = row * LANES + lane;
            double v;
            int j_slot = 0;
            if (what == 2) {
                v = slot_be[sidx];
            } else {
                const int32_t ej = slot_ej[sidx];
                const int64_t e = ej & ID_MASK, j = (uint32_t)ej >> J_SHIFT;
                j_slot = (int)j;
                v = what == 0 ? b_e[j * n_e + e]
                              : reinterpret_cast<const double *>(slot + row * rowb)[j * LANES + lane];
            }
            if (what == 3) {  // spectrum.py:118-120: per-j bincounts, then added j = 0, 1, ..
                if (j_slot != cur_j) {
                    if (cur_j >= 0) s = s + grp;
                    grp = 0.0;
                    cur_j = j_slot;
                }
                grp = grp + v;
            } else {
                s = s + v;
            }
        }
        if (what == 3 && cur_j >= 0) s = s + grp;
        if (old_of_new) out[old_of_new[m]] = s;
        else out[m] = s;
    }
}

__global__ void k_set_free(int64_t n_n, uint8_t *__restrict__ free_int) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_n;
         m += (int64_t)gridDim.x * blockDim.x)
        free_int[m] = 1;
}

__global__ void k_clear_free(int64_t n_d, const int64_t *__restrict__ nd, int64_t n_n,
                             const int32_t *__restrict__ new_of_old, uint8_t *__restrict__ free_int,
                             int32_t *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_d;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t n = nd[i];
        if (n < 0 || n >= n_n) { atomicOr(bad, 1); continue; }
        free_int[new_of_old[n]] = 0;
    }
}

void slot_sum(const Plan *p, int what, const double *b_e, const int32_t *old_of_new, double *out,
              cudaStream_t s) {
    if (p->n_n == 0) return;
    k_slot_sum<<<grid_for(p->n_chunks * LANES, 256), 256, 0, s>>>(
        p->nb, p->n_n, p->n_e, p->rowbase, p->width, p->cnt, p->slot_ej, p->slot, p->rowb, p->slot_be,
        b_e, what, old_of_new, out);
    LAUNCHED();
}

// -------------------------------------------------------------- host helpers --
template <class T>
T read1(const T *dptr, cudaStream_t s) {
    T v;
    CU(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    return v;
}

// exclusive scan of n int32 values; returns the total
static int64_t scan_i32(const int32_t *in, int32_t *out, int64_t n, cudaStream_t s) {
    if (n == 0) return 0;
    size_t bytes = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    void *tmp = dmalloc<char>(bytes);
    cudaError_t err = cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, s);
    cudaFree(tmp);
    CU(err);
    bump_launches(1);
    int32_t last_in = read1(in + n - 1, s), last_out = read1(out + n - 1, s);
    return (int64_t)last_in + last_out;
}

double *plan_vec(Plan *p, int i) {
    if (!p->wvec[i]) p->wvec[i] = dmalloc<double>(p->n_n + 1);
    return p->wvec[i];
}

static void plan_free(Plan *p) {
    dfree(p->new_of_old); dfree(p->old_of_new); dfree(p->cnt); dfree(p->cnt8); dfree(p->codes); dfree(p->tup); dfree(p->rowbase);
    dfree(p->width); dfree(p->slot_ej); dfree(p->slot); dfree(p->tab); dfree(p->taboff);
    dfree(p->slot_be); dfree(p->b_int); dfree(p->free_int); dfree(p->partials);
    dfree(p->ctl); dfree(p->hist_dev); dfree(p->flag); dfree(p->nf_state); dfree(p->rowflag);
    for (auto &v : p->wvec) dfree(v);
    perm_free(p);
    dist_free(p);
    hostpipe_free(p);
    many_free(p);
    if (p->ctl_host) cudaFreeHost(p->ctl_host);
    p->ctl_host = nullptr;
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    p->cap_stream = nullptr;
    if (p->order.ev) cudaEventDestroy(p->order.ev);
    p->order.ev = nullptr;
    for (auto &e : p->ring_ev) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
    }
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_plan_create(int nb, int64_t n_n, int64_t n_e, const int32_t *conn, void *stream,
                    ebs_plan_t *out) {
    Plan *p = nullptr;
    int32_t *cnt_old = nullptr, *flag = nullptr, *pos = nullptr, *iso = nullptr,
            *rowptr = nullptr, *fill = nullptr, *bad = nullptr;
    unsigned long long *first = nullptr;
    int64_t *keys = nullptr;
    EBS_TRY
    EBS_REQUIRE(out, "out must not be NULL");
    *out = nullptr;
    EBS_REQUIRE(nb == 3 || nb == 4, "nb must be 3 (triangles) or 4 (tetrahedra), got %d", nb);
    EBS_REQUIRE(n_n >= 0 && n_e >= 0, "negative sizes");
    EBS_REQUIRE(n_n < (int64_t)ID_MASK && n_e < (int64_t)ID_MASK,
                "mesh too large: need n_nodes, n_elems < 2^30");
    EBS_REQUIRE((int64_t)nb * n_e < (1ll << 31) - 1, "too many element slots (nb*n_e >= 2^31)");
    cudaStream_t s = S(stream);
    p = new Plan();
    p->nb = nb;
    p->n_n = n_n;
    p->n_e = n_e;
    p->n_chunks = (n_n + LANES - 1) / LANES;
    p->flag = dmalloc<int32_t>(4);
    p->nf_state = dmalloc<int32_t>(2 * MANY_MAX);  // one pair per stream of ebs_residual_many
    CU(cudaMemsetAsync(p->nf_state, 0, 2 * MANY_MAX * sizeof(int32_t), s));
    const int64_t total = (int64_t)nb * n_e;

    // 1. valence + first appearance
    cnt_old = dmalloc<int32_t>(n_n);
    first = dmalloc<unsigned long long>(n_n);
    bad = dmalloc<int32_t>(1);
    CU(cudaMemsetAsync(cnt_old, 0, sizeof(int32_t) * (n_n ? n_n : 1), s));
    CU(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long) * (n_n ? n_n : 1), s));
    CU(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
    if (total) {
        k_incidence<<<grid_for(total, 256), 256, 0, s>>>(nb, n_n, n_e, conn, cnt_old, first, bad);
        LAUNCHED();
    }
    EBS_REQUIRE(read1(bad, s) == 0, "element connectivity references nonexistent nodes");

    // 2. internal numbering: the caller's own when it is a structured grid (every id
    // difference a combination of axis strides; sell.cuh IDS_TUPLE), else first appearance
    p->new_of_old = dmalloc<int32_t>(n_n);
    p->old_of_new = dmalloc<int32_t>(n_n);
    if (grid_enabled() && total) {
        int32_t *set = dmalloc<int32_t>(DIFF_CAP + 1);
        int32_t h[DIFF_CAP + 1];
        for (int i = 0; i < DIFF_CAP; ++i) h[i] = DIFF_EMPTY;
        h[DIFF_CAP] = 0;
        CU(cudaMemcpyAsync(set, h, sizeof h, cudaMemcpyHostToDevice, s));
        k_diff_set<<<grid_for(n_e, 256, sm_count() * 8), 256, 0, s>>>(nb, n_e, conn, set,
                                                                      set + DIFF_CAP);
        LAUNCHED();
        cudaError_t e1 = cudaMemcpyAsync(h, set, sizeof h, cudaMemcpyDeviceToHost, s);
        cudaError_t e2 = cudaStreamSynchronize(s);
        cudaFree(set);
        CU(e1);
        CU(e2);
        if (!h[DIFF_CAP]) {
            std::vector<int32_t> a;
            for (int i = 0; i < DIFF_CAP; ++i)
                if (h[i] != DIFF_EMPTY) a.push_back(h[i]);
            std::sort(a.begin(), a.end());
            a.erase(std::unique(a.begin(), a.end()), a.end());
            p->identity = find_strides(nb - 1, a, p->stride);
        }
    }
    if (p->identity && n_n) {
        k_iota<<<grid_for(n_n, 256), 256, 0, s>>>(n_n, p->new_of_old, p->old_of_new);
        LAUNCHED();
    }
    flag = dmalloc<int32_t>(total);
    pos = dmalloc<int32_t>(total);
    int64_t n_conn = 0;
    if (total) {
        k_first_flags<<<grid_for(total, 256), 256, 0, s>>>(nb, n_e, conn, first, flag);
        LAUNCHED();
        n_conn = scan_i32(flag, pos, total, s);
    }
    iso = dmalloc<int32_t>(n_n);
    int32_t *iso_pos = dmalloc<int32_t>(n_n);
    if (n_n) {
        k_isolated_flags<<<grid_for(n_n, 256), 256, 0, s>>>(n_n, cnt_old, iso);
        LAUNCHED();
        scan_i32(iso, iso_pos, n_n, s);
        if (!p->identity) {
            k_numbering<<<grid_for(n_n, 256), 256, 0, s>>>(n_n, n_conn, cnt_old, first, pos,
                                                          iso_pos, p->new_of_old, p->old_of_new);
            LAUNCHED();
        }
    }
    cudaFree(iso_pos);
    dfree(flag);
    dfree(pos);
    dfree(iso);

    // 3. incidence CSR in internal numbering, keys sorted per node
    p->cnt = dmalloc<int32_t>(n_n);
    rowptr = dmalloc<int32_t>(n_n);
    if (n_n) {
        k_permute_cnt<<<grid_for(n_n, 256), 256, 0, s>>>(n_n, p->old_of_new, cnt_old, p->cnt);
        LAUNCHED();
        scan_i32(p->cnt, rowptr, n_n, s);
    }
    keys = dmalloc<int64_t>(total);
    fill = dmalloc<int32_t>(n_n);
    CU(cudaMemsetAsync(fill, 0, sizeof(int32_t) * (n_n ? n_n : 1), s));
    if (total) {
        k_fill_keys<<<grid_for(total, 256), 256, 0, s>>>(nb, n_e, conn, p->new_of_old, rowptr,
                                                        fill, keys);
        LAUNCHED();
        k_sort_segments<<<grid_for(n_n, 128), 128, 0, s>>>(n_n, rowptr, p->cnt, keys);
        LAUNCHED();
    }
    dfree(fill);

    // 4. SELL-32 chunks
    p->width = dmalloc<int32_t>(p->n_chunks);
    p->rowbase = dmalloc<int32_t>(p->n_chunks);
    p->n_rows = 0;
    if (p->n_chunks) {
        k_chunk_width<<<grid_for(p->n_chunks, 256), 256, 0, s>>>(n_n, p->n_chunks, p->cnt,
                                                                p->width);
        LAUNCHED();
        p->n_rows = scan_i32(p->width, p->rowbase, p->n_chunks, s);
    }
    EBS_REQUIRE(p->n_rows * LANES * (int64_t)nb < (1ll << 40), "slot stream too large");
    p->slot_ej = dmalloc<int32_t>(p->n_rows * LANES);
    {
        int32_t *ids_abs = dmalloc<int32_t>(p->n_rows * LANES * (nb - 1));
        unsigned long long *md = dmalloc<unsigned long long>(1);
        CU(cudaMemsetAsync(md, 0, sizeof(unsigned long long), s));
        if (p->n_chunks) {
            k_fill_slots<<<grid_for(p->n_chunks * LANES, 128), 128, 0, s>>>(
                nb, n_n, n_e, conn, p->new_of_old, rowptr, p->cnt, keys, p->rowbase, p->width,
                p->slot_ej, ids_abs, md);
            LAUNCHED();
        }
        unsigned long long max_delta = read1(md, s);
        cudaFree(md);
        // id layout: per-chunk delta tables when every chunk has few distinct deltas,
        // else packed deltas (2 x 15 bit 2D / 3 x 20 bit 3D, biased), else absolute ids
        const int cap = nb == 3 ? 128 : 256;
        int layout = -1;
        int32_t *counts = nullptr;
        if (EBS_IDS_TABLE && p->n_chunks) {
            counts = dmalloc<int32_t>(p->n_chunks);
            CU(cudaMemsetAsync(p->flag, 0, sizeof(int32_t), s));
            k_chunk_tables<<<grid_for(p->n_chunks * 32, 128, sm_count() * 16), 128, 0, s>>>(
                nb, n_n, p->n_chunks, cap, p->rowbase, p->width, p->cnt, ids_abs, counts, nullptr,
                nullptr, nullptr, 0, p->flag);
            LAUNCHED();
            if (read1(p->flag, s) == 0) layout = 2;
        }
        const unsigned long long limit = nb == 3 ? (1ull << 14) - 1 : (1ull << 19) - 1;
        // structured caller numbering: one-byte tuple codes where they measured faster
        std::vector<unsigned long long> tkeys;
        if (p->identity && tuple_wanted(nb, n_n) && max_delta < (1ull << 19) && p->n_chunks) {
            unsigned long long *set = dmalloc<unsigned long long>(TUPLE_CAP + 1);
            std::vector<unsigned long long> h(TUPLE_CAP + 1, TUP_EMPTY);
            h[TUPLE_CAP] = 0;
            CU(cudaMemcpyAsync(set, h.data(), sizeof(unsigned long long) * (TUPLE_CAP + 1),
                               cudaMemcpyHostToDevice, s));
            k_tuple_set<<<grid_for(n_n, 256, sm_count() * 8), 256, 0, s>>>(
                nb, n_n, p->n_chunks, p->rowbase, p->cnt, ids_abs, set,
                reinterpret_cast<int32_t *>(set + TUPLE_CAP));
            LAUNCHED();
            cudaError_t e1 = cudaMemcpyAsync(h.data(), set, sizeof(unsigned long long) * (TUPLE_CAP + 1),
                                             cudaMemcpyDeviceToHost, s);
            cudaError_t e2 = cudaStreamSynchronize(s);
            cudaFree(set);
            CU(e1);
            CU(e2);
            if (h[TUPLE_CAP] == 0) {
                for (int i = 0; i < TUPLE_CAP; ++i)
                    if (h[i] != TUP_EMPTY) tkeys.push_back(h[i]);
                std::sort(tkeys.begin(), tkeys.end());
                tkeys.erase(std::unique(tkeys.begin(), tkeys.end()), tkeys.end());
                if (!tkeys.empty()) layout = IDS_TUPLE;
            }
        }
        if (layout < 0) layout = max_delta <= limit ? 1 : 0;
        if (layout == 1 && nb == 4 && EBS_IDS_DELTA2) layout = 3;  // same plane, two-base rows
        p->packed = layout;
        const int id_bytes = layout == IDS_TUPLE ? 0
                           : layout == 2 ? (nb == 3 ? 2 : 4) * LANES
                                         : (layout == 1 || layout == 3 ? (nb == 3 ? 4 : 8) * LANES
                                                        : 4 * (nb - 1) * LANES);
        p->rowb = nb * 8 * LANES + id_bytes;
        p->slot = dmalloc<uint8_t>((size_t)p->n_rows * p->rowb);
        CU(cudaMemsetAsync(p->slot, 0, (size_t)p->n_rows * p->rowb, s));
        p->taboff = dmalloc<int32_t>(p->n_chunks + 1);
        CU(cudaMemsetAsync(p->taboff, 0, sizeof(int32_t) * (p->n_chunks + 1), s));
        if (layout == 2) {
            const int32_t ntab = (int32_t)scan_i32(counts, p->taboff, p->n_chunks, s);
            CU(cudaMemcpyAsync(p->taboff + p->n_chunks, &ntab, sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
            CU(cudaStreamSynchronize(s));
            p->tab = dmalloc<int32_t>(ntab);
            k_chunk_tables<<<grid_for(p->n_chunks * 32, 128, sm_count() * 16), 128, 0, s>>>(
                nb, n_n, p->n_chunks, cap, p->rowbase, p->width, p->cnt, ids_abs, nullptr,
                p->taboff, p->tab, p->slot, p->rowb, p->flag);
            LAUNCHED();
        } else if (layout == IDS_TUPLE) {
            p->tab = dmalloc<int32_t>(1);
            const int nk = (int)tkeys.size();
            std::vector<int4> tab(TUPLE_CAP, make_int4(0, 0, 0, 0));
            for (int i = 0; i < nk; ++i) {
                const unsigned long long k = tkeys[i];
                int d[3] = {0, 0, 0};
                for (int t = 0; t < nb - 1; ++t)
                    d[t] = (int)((k >> (20 * t)) & 0xFFFFF) - (1 << 19);
                tab[i] = make_int4((int)(k >> 60), d[0], d[1], d[2]);
            }
            p->n_tup = nk;
            p->tup = dmalloc<int4>(TUPLE_CAP);
            CU(cudaMemcpyAsync(p->tup, tab.data(), sizeof(int4) * TUPLE_CAP, cudaMemcpyHostToDevice, s));
            unsigned long long *dk = dmalloc<unsigned long long>(nk);
            CU(cudaMemcpyAsync(dk, tkeys.data(), sizeof(unsigned long long) * nk, cudaMemcpyHostToDevice, s));
            p->codes = dmalloc<uint8_t>((size_t)p->n_rows * LANES);
            CU(cudaMemsetAsync(p->flag, 0, sizeof(int32_t), s));
            k_write_codes<<<grid_for(p->n_chunks * LANES, 128), 128, 0, s>>>(
                nb, n_n, p->n_chunks, p->rowbase, p->width, p->cnt, ids_abs, dk, nk, p->codes,
                p->flag);
            LAUNCHED();
            const int32_t bad_code = read1(p->flag, s);
            cudaFree(dk);
            EBS_REQUIRE(bad_code == 0, "internal error: slot tuple missing from the table");
        } else if (layout == 3 && p->n_chunks) {
            p->tab = dmalloc<int32_t>(1);
            p->rowflag = dmalloc<uint8_t>(p->n_rows);
            unsigned long long *nt = dmalloc<unsigned long long>(1);
            CU(cudaMemsetAsync(nt, 0, sizeof(unsigned long long), s));
            k_write_ids_delta2<<<grid_for(p->n_chunks * LANES, 128), 128, 0, s>>>(
                n_n, p->n_chunks, p->rowb, p->rowbase, p->width, p->cnt, ids_abs, p->slot,
                p->rowflag, nt);
            LAUNCHED();
            unsigned long long h = 0;
            CU(cudaMemcpyAsync(&h, nt, sizeof h, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            cudaFree(nt);
            p->two_base_rows = (int64_t)h;
        } else if (p->n_chunks) {
            p->tab = dmalloc<int32_t>(1);
            k_write_ids<<<grid_for(p->n_chunks * LANES, 128), 128, 0, s>>>(
                nb, n_n, p->n_chunks, p->rowb, p->packed, p->rowbase, p->width, ids_abs, p->slot);
            LAUNCHED();
        }
        if (counts) cudaFree(counts);
        CU(cudaStreamSynchronize(s));
        cudaFree(ids_abs);
    }
    // max valence (for info)
    {
        int32_t mv = 0;
        if (p->n_chunks) {
            int32_t *w = new int32_t[p->n_chunks];
            cudaError_t e1 = cudaMemcpyAsync(w, p->width, sizeof(int32_t) * p->n_chunks,
                                             cudaMemcpyDeviceToHost, s);
            cudaError_t e2 = cudaStreamSynchronize(s);
            for (int64_t c = 0; c < p->n_chunks; ++c) mv = w[c] > mv ? w[c] : mv;
            delete[] w;
            CU(e1);
            CU(e2);
        }
        p->max_valence = mv;
    }
    // one-byte valences for the sweeps (C2: 4.2 MB instead of 16.8 MB per pass)
    if (p->max_valence <= 255 && n_n > 0) {
        p->cnt8 = dmalloc<uint8_t>(n_n);
        k_cnt8<<<grid_for(n_n, 256), 256, 0, s>>>(n_n, p->cnt, p->cnt8);
        LAUNCHED();
    }
    dfree(keys);
    dfree(rowptr);
    dfree(cnt_old);
    dfree(first);
    dfree(bad);

    // control block + reduction scratch
    p->ctl = dmalloc<Ctl>(1);
    CU(cudaMemsetAsync(p->ctl, 0, sizeof(Ctl), s));
    CU(cudaMallocHost(&p->ctl_host, 3 * sizeof(Ctl)));  // [0] synchronous reads, [1..2] ring
    p->partials = dmalloc<double>(4 * 8192);
    p->free_int = dmalloc<uint8_t>(n_n);
    if (n_n) {
        k_set_free<<<grid_for(n_n, 256), 256, 0, s>>>(n_n, p->free_int);
        LAUNCHED();
    }
    CU(cudaStreamSynchronize(s));
    *out = reinterpret_cast<ebs_plan_t>(p);
    p = nullptr;
    }
    catch (const ebs::Fail &f) {
        cudaFree(cnt_old); cudaFree(flag); cudaFree(pos); cudaFree(iso); cudaFree(rowptr);
        cudaFree(fill); cudaFree(bad); cudaFree(first); cudaFree(keys);
        if (p) { plan_free(p); delete p; }
        return f.code;
    }
    catch (...) {
        if (p) { plan_free(p); delete p; }
        set_error("unexpected C++ exception in ebs_plan_create");
        return EBS_ECUDA;
    }
    return EBS_OK;
}

int ebs_plan_destroy(ebs_plan_t plan) {
    if (!plan) return EBS_OK;
    Plan *p = reinterpret_cast<Plan *>(plan);
    plan_free(p);
    delete p;
    return EBS_OK;
}

int ebs_plan_info(ebs_plan_t plan, int64_t *info) {
    EBS_TRY
    EBS_REQUIRE(plan && info, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    info[0] = p->n_n;
    info[1] = p->n_e;
    info[2] = p->nb;
    info[3] = p->n_chunks;
    info[4] = p->n_rows;
    int64_t slots = p->n_rows * LANES;
    info[5] = p->n_rows * (int64_t)p->rowb + (p->has_be ? slots * 8 : 0) + (p->codes ? slots : 0);
    info[6] = p->max_valence;
    info[7] = (p->has_A ? 1 : 0) | (p->has_be ? 2 : 0) | (p->packed ? 4 : 0) |
              (p->packed == 2 ? 8 : 0) | (p->packed == 3 ? 16 : 0) |
              (p->packed == IDS_TUPLE ? 32 : 0) | (p->identity ? 64 : 0);
    EBS_CATCH
}

int ebs_plan_node_maps(ebs_plan_t plan, int32_t *new_of_old, int32_t *old_of_new,
                       void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan, "null plan");
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (p->n_n == 0) return EBS_OK;
    if (new_of_old)
        CU(cudaMemcpyAsync(new_of_old, p->new_of_old, sizeof(int32_t) * p->n_n,
                           cudaMemcpyDeviceToDevice, S(stream)));
    if (old_of_new)
        CU(cudaMemcpyAsync(old_of_new, p->old_of_new, sizeof(int32_t) * p->n_n,
                           cudaMemcpyDeviceToDevice, S(stream)));
    EBS_CATCH
}

int ebs_plan_load(ebs_plan_t plan, const double *A_e, const double *b_e, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan, "null plan");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(A_e || p->n_e == 0, "null A_e");
    cudaStream_t s = S(stream);
    OrderGuard order(p->order, s);
    const int64_t n_slots = p->n_rows * LANES;
    const bool want_be = b_e != nullptr || p->n_e == 0;  // an empty mesh has an (empty) b_e
    if (want_be && !p->slot_be) p->slot_be = dmalloc<double>(n_slots);
    if (want_be && !p->b_int) p->b_int = dmalloc<double>(p->n_n);
    if (n_slots) {
        k_pack<<<grid_for(n_slots, 256, sm_count() * 64), 256, 0, s>>>(
            p->nb, p->n_e, n_slots, p->rowb, p->slot_ej, A_e, b_e, p->slot,
            b_e ? p->slot_be : nullptr);
        LAUNCHED();
    }
    p->has_A = 1;
    p->has_be = want_be ? 1 : 0;
    if (want_be && p->n_n) {
        k_slot_sum<<<grid_for(p->n_chunks * LANES, 256), 256, 0, s>>>(
            p->nb, p->n_n, p->n_e, p->rowbase, p->width, p->cnt, p->slot_ej, p->slot, p->rowb,
            p->slot_be, nullptr, 2, nullptr, p->b_int);
        LAUNCHED();
    }
    EBS_CATCH
}

int ebs_plan_set_dirichlet(ebs_plan_t plan, const int64_t *nd, int64_t n_d, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && n_d >= 0, "bad arguments");
    Plan *p = reinterpret_cast<Plan *>(plan);
    cudaStream_t s = S(stream);
    OrderGuard order(p->order, s);
    if (p->n_n) {
        k_set_free<<<grid_for(p->n_n, 256), 256, 0, s>>>(p->n_n, p->free_int);
        LAUNCHED();
    }
    p->n_dirichlet = n_d;
    if (n_d) {
        CU(cudaMemsetAsync(p->flag, 0, sizeof(int32_t), s));
        k_clear_free<<<grid_for(n_d, 256), 256, 0, s>>>(n_d, nd, p->n_n, p->new_of_old,
                                                       p->free_int, p->flag);
        LAUNCHED();
        EBS_REQUIRE(read1(p->flag, s) == 0, "Dirichlet node index out of range");
    }
    EBS_CATCH
}

int ebs_assemble_rhs(ebs_plan_t plan, const double *b_e, double *b, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && b_e && b, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (p->n_n == 0) return EBS_OK;
    k_slot_sum<<<grid_for(p->n_chunks * LANES, 256), 256, 0, S(stream)>>>(
        p->nb, p->n_n, p->n_e, p->rowbase, p->width, p->cnt, p->slot_ej, nullptr, 0, nullptr, b_e,
        0, p->old_of_new, b);
    LAUNCHED();
    EBS_CATCH
}

int ebs_diagonal(ebs_plan_t plan, double *d, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && d, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    if (p->n_n == 0) return EBS_OK;
    k_slot_sum<<<grid_for(p->n_chunks * LANES, 256), 256, 0, S(stream)>>>(
        p->nb, p->n_n, p->n_e, p->rowbase, p->width, p->cnt, p->slot_ej, p->slot, p->rowb, nullptr,
        nullptr, 1, p->old_of_new, d);
    LAUNCHED();
    EBS_CATCH
}

int ebs_plan_internal_diag(ebs_plan_t plan, double *d_int, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && d_int, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    slot_sum(p, 1, nullptr, nullptr, d_int, S(stream));
    EBS_CATCH
}

int ebs_diagonal_grouped(ebs_plan_t plan, double *d, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && d, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    slot_sum(p, 3, nullptr, p->old_of_new, d, S(stream));
    EBS_CATCH
}

}  // extern "C"

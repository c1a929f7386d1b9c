// perm.cu -- caller <-> internal node permutation with every global access coalesced.
//
// Why: the caller's node numbering may be an arbitrary permutation of the plan's internal
// (first-appearance) numbering (BASELINE C2).  A direct gather y[m] = x[old_of_new[m]]
// touches 32 distinct 128 B lines per warp instruction; the L1tex pipe processes one line
// per ~2 cycles, so 4.2M random 8 B accesses cost ~30 us at C2 no matter how many loads
// are in flight (ncu: lg_throttle + long-scoreboard, DRAM at 23%).  Here the permutation
// runs in two passes through shared memory:
//
//   pass 1 (one CTA per source tile of T nodes): load the tile coalesced into smem, then
//          write it out in destination-bucket order: inter[dst1[q]] = tile[src1[q]] --
//          consecutive q of a tile land in contiguous runs of ~T/n_tiles values.
//   pass 2 (one CTA per destination tile):  read inter[bT .. bT+T) coalesced, place each
//          value at its offset dst2[k] inside the tile in smem, write the tile coalesced.
//
// The schedule (src1 u16, dst1 i32, dst2 u16: 8 B per node and direction) is built once
// per plan on the device with two stable radix sorts.  Values are moved, never combined:
// results are bit-identical to the direct gather.
#include <cub/cub.cuh>

#include "ebs_internal.cuh"

namespace ebs {

#ifndef EBS_PERM_SEG
#define EBS_PERM_SEG 16  // target run length (values) of the pass-1 writes: T*T >= SEG*n
#endif

// tile size: the smallest power of two in [2048, 16384] whose pass-1 runs (T*T/n values
// on average) reach EBS_PERM_SEG -- the run length is what coalesces the pass-1 stores
static int perm_tile(int64_t n) {
    int T = 2048;
    while (T < 16384 && (int64_t)T * T < (int64_t)EBS_PERM_SEG * n) T *= 2;
    return T;
}

__global__ void k_perm_keys(int64_t n, int T, const int32_t *__restrict__ dest,
                            int32_t *__restrict__ key, int32_t *__restrict__ val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = dest[i] / T;
        val[i] = (int32_t)i;
    }
}

// order[k] = source of intermediate slot k (sorted by destination tile, then source)
__global__ void k_perm_stage2(int64_t n, int T, const int32_t *__restrict__ dest,
                              const int32_t *__restrict__ order, uint16_t *__restrict__ dst2,
                              int32_t *__restrict__ key, int32_t *__restrict__ val) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = order[k];
        dst2[k] = (uint16_t)(dest[i] - (k / T) * T);
        key[k] = i / T;  // source tile
        val[k] = (int32_t)k;
    }
}

// dst1[q] = intermediate slot of the q-th value written by its source tile (the second
// sort's output); src1[q] = that value's offset inside the source tile
__global__ void k_perm_stage3(int64_t n, int T, const int32_t *__restrict__ order,
                              const int32_t *__restrict__ dst1, uint16_t *__restrict__ src1) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        src1[q] = (uint16_t)(order[dst1[q]] - (q / T) * T);
}

// one CTA per tile; every thread issues its PE loads back to back (latency overlap)
template <int T, int TH>
__global__ void __launch_bounds__(TH)
    k_perm_pass1(int64_t n, const double *__restrict__ x, const uint16_t *__restrict__ src1,
                 const int32_t *__restrict__ dst1, double *__restrict__ inter,
                 int32_t *nonfinite) {
    constexpr int PE = T / TH;
    extern __shared__ double tile[];
    const int64_t base = (int64_t)blockIdx.x * T;
    const int cnt = n - base < T ? (int)(n - base) : T;
    double v[PE];
#pragma unroll
    for (int u = 0; u < PE; ++u) {
        const int t = threadIdx.x + u * TH;
        v[u] = t < cnt ? __ldcs(x + base + t) : 0.0;
    }
    int32_t d[PE];
    uint16_t sidx[PE];
#pragma unroll
    for (int u = 0; u < PE; ++u) {
        const int q = threadIdx.x + u * TH;
        d[u] = q < cnt ? __ldcs(dst1 + base + q) : 0;
        sidx[u] = q < cnt ? __ldcs(src1 + base + q) : 0;
    }
    bool bad = false;
#pragma unroll
    for (int u = 0; u < PE; ++u) {
        tile[threadIdx.x + u * TH] = v[u];
        bad |= !isfinite(v[u]);
    }
    if (__syncthreads_or(bad) && nonfinite && threadIdx.x == 0) atomicOr(nonfinite, 1);
#pragma unroll
    for (int u = 0; u < PE; ++u)
        if (threadIdx.x + u * TH < cnt) inter[d[u]] = tile[sidx[u]];
}

template <int T, int TH>
__global__ void __launch_bounds__(TH)
    k_perm_pass2(int64_t n, const double *__restrict__ inter, const uint16_t *__restrict__ dst2,
                 double *__restrict__ out) {
    constexpr int PE = T / TH;
    extern __shared__ double tile[];
    const int64_t base = (int64_t)blockIdx.x * T;
    const int cnt = n - base < T ? (int)(n - base) : T;
    double v[PE];
    uint16_t d[PE];
#pragma unroll
    for (int u = 0; u < PE; ++u) {
        const int k = threadIdx.x + u * TH;
        v[u] = k < cnt ? __ldcs(inter + base + k) : 0.0;
        d[u] = k < cnt ? __ldcs(dst2 + base + k) : 0;
    }
#pragma unroll
    for (int u = 0; u < PE; ++u)
        if (threadIdx.x + u * TH < cnt) tile[d[u]] = v[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PE; ++u) {
        const int t = threadIdx.x + u * TH;
        if (t < cnt) out[base + t] = tile[t];
    }
}

static void build(Perm2 &P, int64_t n, const int32_t *dest, cudaStream_t s) {
    const int T = perm_tile(n);
    P.n = n;
    P.T = T;
    P.src1 = dmalloc<uint16_t>(n);
    P.dst1 = dmalloc<int32_t>(n);
    P.dst2 = dmalloc<uint16_t>(n);
    const int64_t tiles = (n + T - 1) / T;
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < tiles) ++end_bit;
    int32_t *k0 = dmalloc<int32_t>(n), *k1 = dmalloc<int32_t>(n);
    int32_t *v0 = dmalloc<int32_t>(n), *v1 = dmalloc<int32_t>(n);
    size_t bytes = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, v0, v1, (int)n, 0, end_bit, s));
    char *tmp = dmalloc<char>(bytes);
    const int g = grid_for(n, 256);
    k_perm_keys<<<g, 256, 0, s>>>(n, T, dest, k0, v0);
    LAUNCHED();
    CU(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, v1, (int)n, 0, end_bit, s));
    bump_launches(1);
    // v1 = order; reuse k0/v0 for the second sort's input
    k_perm_stage2<<<g, 256, 0, s>>>(n, T, dest, v1, P.dst2, k0, v0);
    LAUNCHED();
    CU(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, v0, P.dst1, (int)n, 0, end_bit, s));
    bump_launches(1);
    k_perm_stage3<<<g, 256, 0, s>>>(n, T, v1, P.dst1, P.src1);
    LAUNCHED();
    CU(cudaStreamSynchronize(s));
    cudaFree(tmp);
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1);
}

template <int T, int TH>
static void launch_passes(const Perm2 *P, const double *in, double *out, double *inter,
                          int32_t *nonfinite, cudaStream_t s) {
    static bool attr[64] = {};  // dynamic smem above 48 KB: opt-in per kernel and device
    int dev = 0;
    CU(cudaGetDevice(&dev));
    if (!attr[dev & 63]) {
        CU(cudaFuncSetAttribute(k_perm_pass1<T, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                T * 8));
        CU(cudaFuncSetAttribute(k_perm_pass2<T, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                T * 8));
        attr[dev & 63] = true;
    }
    const int tiles = (int)((P->n + T - 1) / T);
    k_perm_pass1<T, TH><<<tiles, TH, T * 8, s>>>(P->n, in, P->src1, P->dst1, inter, nonfinite);
    LAUNCHED();
    k_perm_pass2<T, TH><<<tiles, TH, T * 8, s>>>(P->n, inter, P->dst2, out);
    LAUNCHED();
}

// the schedule of direction dir (0: caller -> internal, 1: internal -> caller), built on
// first use; nullptr when it cannot be built now (stream capture in progress)
const Perm2 *perm_get(Plan *p, int dir, cudaStream_t s) {
    Perm2 &P = p->perm[dir];
    if (P.src1) return &P;
    if (p->n_n == 0 || p->n_n >= (int64_t(1) << 31)) return nullptr;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(s, &st));
    if (st != cudaStreamCaptureStatusNone) return nullptr;
    plan_vec(p, PERM_VEC);  // allocate the intermediate now (not during a capture)
    try {
        build(P, p->n_n, dir == 0 ? p->new_of_old : p->old_of_new, s);
    } catch (...) {
        dfree(P.src1); dfree(P.dst1); dfree(P.dst2);
        throw;
    }
    return &P;
}

void perm_apply(Plan *p, const Perm2 *P, const double *in, double *out, int32_t *nonfinite,
                cudaStream_t s) {
    double *inter = plan_vec(p, PERM_VEC);
    switch (P->T) {
        case 2048: launch_passes<2048, 256>(P, in, out, inter, nonfinite, s); break;
        case 4096: launch_passes<4096, 512>(P, in, out, inter, nonfinite, s); break;
        case 8192: launch_passes<8192, 1024>(P, in, out, inter, nonfinite, s); break;
        default: launch_passes<16384, 1024>(P, in, out, inter, nonfinite, s); break;
    }
}

void perm_free(Plan *p) {
    for (auto &P : p->perm) { dfree(P.src1); dfree(P.dst1); dfree(P.dst2); }
}

}  // namespace ebs

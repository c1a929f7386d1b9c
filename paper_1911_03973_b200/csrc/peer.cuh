// peer.cuh -- window layout and synchronisation primitives of the peer-memory halo and
// all-reduce (peer.cu; the fused all-reduce consumer in dist.cu's single-reduction PCG step).
#pragma once
#include "ebs_internal.cuh"

namespace ebs {

constexpr int PEER_MAX = EBS_PEER_MAX;   // ranks per peer group (one NVSwitch node)
constexpr int PEER_RED_MAX = 256;        // doubles per all-reduce launch

struct WinHdr {
    unsigned long long halo_flag[PEER_MAX];  // [src]: last halo epoch + 1 that src published
    unsigned long long red_flag[PEER_MAX];   // [src]: the same for the all-reduce slots
    unsigned long long halo_epoch;           // local: halo exchanges completed
    unsigned long long red_epoch;            // local: all-reduces completed
    unsigned int arrive;                     // interface chunks / blocks done (running put)
    unsigned int error;                      // 1: a wait timed out
    unsigned int done_a;                     // k_peer_jacobi_step: completion warps done
    unsigned int pad[25];
};
static_assert(sizeof(WinHdr) == 256, "window header is 256 bytes");
constexpr size_t RED_OFF = 256;
constexpr size_t RECV_OFF = RED_OFF + sizeof(double) * 2 * PEER_MAX * PEER_RED_MAX;

inline size_t window_bytes(int64_t cap) {
    return RECV_OFF + sizeof(double) * (size_t)PEER_MAX * 2 * (size_t)cap;
}
__host__ __device__ inline double *win_red(char *win, int parity, int src) {
    return reinterpret_cast<double *>(win + RED_OFF) + ((size_t)parity * PEER_MAX + src) * PEER_RED_MAX;
}
__host__ __device__ inline double *win_recv(char *win, int64_t cap, int src, int parity) {
    return reinterpret_cast<double *>(win + RECV_OFF) + ((size_t)src * 2 + parity) * cap;
}

// ------------------------------------------------------------- sync primitives --
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// a flag store after an explicit __threadfence_system() (fence.sc.sys + relaxed store =
// release): one fence for all the flags of a publish instead of one per st.release
__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    return *reinterpret_cast<const volatile unsigned long long *>(p);
}
__device__ __forceinline__ long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (long long)t;
}

// wait until *flag >= want; false (and the error word set) after timeout_ns
static __device__ __noinline__ bool peer_wait(const unsigned long long *flag, unsigned long long want,
                                       long long timeout_ns, unsigned int *err) {
    if (ld_acquire_sys(flag) >= want) return true;
    const long long t0 = global_ns();
    unsigned ns = 32;
    while (ld_acquire_sys(flag) < want) {
        if (*reinterpret_cast<volatile unsigned int *>(err)) return false;
        __nanosleep(ns);
        if (ns < 256) ns *= 2;
        if (global_ns() - t0 > timeout_ns) {
            atomicExch(err, 1u);
            return false;
        }
    }
    return true;
}

#ifndef EBS_PEER_BREAK_PARITY
#define EBS_PEER_BREAK_PARITY 0  // negative control of ebs_peer_selftest only (one slot, no
#endif                           // double buffering): must report errors (profiles/)

// The receiving side of a rank's halo (peer.cu builds it from the peer view).
struct PeerRecv {
    WinHdr *hdr;
    const char *win;  // this rank's window
    int64_t cap;
    int64_t n_if;
    const int64_t *all_if;
    const int32_t *pos;
    int n_src;
    int src[PEER_MAX];
    int rank;
    long long timeout_ns;
};

// every block: wait for the neighbours' flags of epoch ep (thread k waits for source k)
__device__ __forceinline__ unsigned long long recv_wait(const PeerRecv &r) {
    const unsigned long long ep = ld_volatile(&r.hdr->halo_epoch);
    if (threadIdx.x < r.n_src && r.src[threadIdx.x] != r.rank)
        peer_wait(&r.hdr->halo_flag[r.src[threadIdx.x]], ep + 1, r.timeout_ns, &r.hdr->error);
    __syncthreads();
    return ep;
}

// sum of the contributions to shared node i in ascending rank order (own partial: v)
__device__ __forceinline__ double recv_sum(const PeerRecv &r, int64_t i, const double *v,
                                           int par) {
    if (EBS_PEER_BREAK_PARITY) par = 0;
    double acc = 0.0;
    for (int k = 0; k < r.n_src; ++k) {
        const int32_t q = r.pos[i * r.n_src + k];
        if (q < 0) continue;
        EBS_DCHECK(r.src[k] == r.rank || q < r.cap);
        acc += r.src[k] == r.rank
                   ? v[q]
                   : __ldcg(win_recv(const_cast<char *>(r.win), r.cap, r.src[k], par) + q);
    }
    return acc;
}

// Fused all-reduce consumer: the ranks' contributions were put into this window's slots
// (ebs_peer_allreduce mode 1, or the put of ebs_peer_combine_q); wait for every rank's flag
// of the current epoch and add the slots in rank order 0..world-1 (identical on every rank).
struct RedGet {
    char *win;   // this rank's window; nullptr: no peer all-reduce (values already reduced)
    int world;
    long long timeout_ns;
};

// every block: v[0..n) = the rank-ordered sums (valid in all threads); returns the epoch
template <int N>
__device__ __forceinline__ unsigned long long red_get_block(const RedGet &g, double (&v)[N]) {
    __shared__ double sv[N];
    WinHdr *h = reinterpret_cast<WinHdr *>(g.win);
    const unsigned long long ep = ld_volatile(&h->red_epoch);
    if (threadIdx.x < g.world) peer_wait(&h->red_flag[threadIdx.x], ep + 1, g.timeout_ns, &h->error);
    __syncthreads();
    const int par = (int)(ep & 1);
    if (threadIdx.x < N) {
        double s = __ldcg(win_red(g.win, par, 0) + threadIdx.x);
        for (int q = 1; q < g.world; ++q) s += __ldcg(win_red(g.win, par, q) + threadIdx.x);
        sv[threadIdx.x] = s;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = sv[i];
    return ep;
}

}  // namespace ebs

// peer.cu -- the element-slab halo exchange and the dot all-reduce over PEER MEMORY
// (SURVEY 8e): each rank owns one device window (cudaMalloc, exported by CUDA IPC and
// mapped by every other rank of the node -- NVLink / NVSwitch P2P on an 8-GPU box); ranks
// write into each other's windows with plain stores and publish with a release store of
// an epoch flag; readers acquire the flag and read their own window.
//
// Hot path (the slab Jacobi / PCG iterations): the SELL sweep over a rank's chunks takes
// the chunks holding interface nodes FIRST; the epilogue of an interface node stores its
// partial sum straight into each sharing neighbour's window, and the last warp to finish
// an interface chunk releases the neighbours' flags -- so the halo travels while the same
// launch sweeps the interior chunks (the exchange overlaps the math chunk by chunk, no
// collective launch, no gather).  The combine kernel that follows acquires the flags,
// sums every shared node over the touching ranks in ascending rank order (own partial
// among them: bitwise the values of the NCCL / device-copy transports) and completes the
// node.  Per rank and iteration: 2 launches (Jacobi), 4 (single-reduction PCG, with the
// all-reduce kernel) instead of 4-7 plus NCCL.
//
// Window layout (bytes): [0, 256) header (flags indexed by SOURCE rank, local epochs,
// arrival counter, error word); [256, 256 + 32 KiB) all-reduce slots [parity][src][256
// doubles]; then the halo slots [src][parity][cap doubles].  Double buffering by epoch
// parity: a sender writes epoch e into slot e & 1 only after completing its own epoch
// e-1 combine, which needed the receiver's epoch e-1 flag, which the receiver set after
// finishing its epoch e-2 read of that slot (stream order) -- so a slot is never
// overwritten while it is read.  Every rank runs the same sequence of exchanges, so
// the local epoch counters agree.  Waits are bounded (globaltimer): on a timeout the
// window's error word is set, the kernel proceeds, and ebs_peer_status reports EBS_ENCCL.
#include "peer.cuh"
#include "sell.cuh"

#include <algorithm>
#include <vector>

namespace ebs {

// ------------------------------------------------------------------ peer state --
struct Peer {
    int rank = 0, world = 1;
    int64_t cap = 0;
    long long timeout_ns = 0;
    char *win[PEER_MAX] = {nullptr};  // mapped windows; win[rank] is this rank's own
    // halo (ebs_peer_set_halo)
    int n_nb = 0;
    int nb[PEER_MAX] = {0};
    int64_t len[PEER_MAX] = {0};
    int64_t n_if = 0;
    int64_t *all_if = nullptr;             // interface nodes (local ids, ascending)
    int32_t *ifx = nullptr;                // [n_local]: position in all_if or -1
    int32_t *snd_off = nullptr;            // [n_if + 1] send entries of interface node i
    unsigned long long *snd_addr = nullptr;  // remote parity-0 slot address per entry
    int32_t *pos = nullptr;                // [n_if][n_src]: index in source k or -1
    int n_src = 0;
    int src[PEER_MAX] = {0};               // combine sources, ascending rank (self included)
    int64_t n_local = 0;
};

WinHdr *hdr_of(const Peer *p) { return reinterpret_cast<WinHdr *>(p->win[p->rank]); }

// ----------------------------------------------------------------- all-reduce --
struct RedArgs {
    char *win[PEER_MAX];
    int rank, world, n;
    long long timeout_ns;
};

// phase 1: this rank's n values into slot [parity][rank] of every window, flags released
__device__ __forceinline__ void red_put(const RedArgs &a, const double *buf, unsigned long long ep) {
    const int par = (int)(ep & 1);
    for (int q = 0; q < a.world; ++q) {
        double *dst = win_red(a.win[q], par, a.rank);
        for (int i = threadIdx.x; i < a.n; i += blockDim.x) dst[i] = buf[i];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // the block's stores (barrier) before the flags
        for (int q = 0; q < a.world; ++q)
            st_relaxed_sys(&reinterpret_cast<WinHdr *>(a.win[q])->red_flag[a.rank], ep + 1);
    }
}

// phase 2: wait for every rank's slot, buf = sum over src = 0..world-1 (fixed order)
__device__ __forceinline__ void red_get(const RedArgs &a, double *buf, unsigned long long ep) {
    WinHdr *h = reinterpret_cast<WinHdr *>(a.win[a.rank]);
    if (threadIdx.x < a.world) peer_wait(&h->red_flag[threadIdx.x], ep + 1, a.timeout_ns, &h->error);
    __syncthreads();
    const int par = (int)(ep & 1);
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
        double s = __ldcg(win_red(a.win[a.rank], par, 0) + i);
        for (int q = 1; q < a.world; ++q) s += __ldcg(win_red(a.win[a.rank], par, q) + i);
        buf[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) h->red_epoch = ep + 1;
}

// mode 0: put + get (one launch, ranks in separate processes); 1: put only; 2: get only
// (ranks emulated in one process: every put is enqueued before any get)
__global__ void __launch_bounds__(256) k_peer_allreduce(__grid_constant__ const RedArgs a,
                                                        double *buf, int mode) {
    WinHdr *h = reinterpret_cast<WinHdr *>(a.win[a.rank]);
    const unsigned long long ep = ld_volatile(&h->red_epoch);
    if (mode != 2) red_put(a, buf, ep);
    if (mode != 1) red_get(a, buf, ep);
}

// --------------------------------------------------------- generic halo put/get --
struct PutArgs {
    WinHdr *hdr;
    int n_nb;
    int64_t off[PEER_MAX + 1];          // prefix of the neighbours' lengths
    const double *src[PEER_MAX];        // per neighbour: len doubles (slot order)
    double *dst[PEER_MAX];              // remote parity-0 slot of this rank in neighbour k
    unsigned long long *flag[PEER_MAX]; // remote halo_flag[rank] of neighbour k
    int64_t cap;
};

__global__ void __launch_bounds__(256) k_peer_put(__grid_constant__ const PutArgs a) {
    const unsigned long long ep = ld_volatile(&a.hdr->halo_epoch);
    const int64_t par = (int64_t)(ep & 1);
    const int64_t tot = a.off[a.n_nb];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (t >= a.off[k + 1]) ++k;
        const int64_t i = t - a.off[k];
        a.dst[k][par * a.cap + i] = a.src[k][i];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&a.hdr->arrive, 1u);
        if (prev == gridDim.x - 1) {
            a.hdr->arrive = 0;
            __threadfence_system();
            for (int k = 0; k < a.n_nb; ++k) st_relaxed_sys(a.flag[k], ep + 1);
        }
    }
}

struct GetArgs {
    WinHdr *hdr;
    int n_nb;
    int nb[PEER_MAX];
    int64_t off[PEER_MAX + 1];
    const double *slot[PEER_MAX];  // local parity-0 slot of neighbour k
    double *out[PEER_MAX];
    int64_t cap;
    long long timeout_ns;
};

__global__ void __launch_bounds__(256) k_peer_get(__grid_constant__ const GetArgs a,
                                                  unsigned int *counter) {
    const unsigned long long ep = ld_volatile(&a.hdr->halo_epoch);
    if (threadIdx.x < a.n_nb)
        peer_wait(&a.hdr->halo_flag[a.nb[threadIdx.x]], ep + 1, a.timeout_ns, &a.hdr->error);
    __syncthreads();
    const int64_t par = (int64_t)(ep & 1);
    const int64_t tot = a.off[a.n_nb];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (t >= a.off[k + 1]) ++k;
        const int64_t i = t - a.off[k];
        a.out[k][i] = __ldcg(a.slot[k] + par * a.cap + i);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        if (prev == gridDim.x - 1) {
            *counter = 0;
            a.hdr->halo_epoch = ep + 1;
        }
    }
}

// ------------------------------------------------------------ fused slab sweeps --
// Interface-node stores of the sweeps: node m's partial s goes to every neighbour that
// shares m, at its slot position (snd_addr: parity-0 address; + parity * cap).
struct PeerSend {
    WinHdr *hdr;
    const int32_t *ifx;
    const int32_t *snd_off;
    const unsigned long long *snd_addr;
    int64_t cap;
    int n_if_chunks;
    int n_nb;
    unsigned long long *flag[PEER_MAX];  // remote halo_flag[rank] of neighbour k
};

__device__ __forceinline__ void peer_push(const PeerSend &ps, int m, double s) {
    const int i = ps.ifx[m];
    const int64_t par =
        EBS_PEER_BREAK_PARITY ? 0 : (int64_t)(ld_volatile(&ps.hdr->halo_epoch) & 1);
    EBS_DCHECK(i >= 0);
    for (int e = ps.snd_off[i]; e < ps.snd_off[i + 1]; ++e)
        reinterpret_cast<double *>(ps.snd_addr[e])[par * ps.cap] = s;
}

// after a warp finished an interface chunk: the last one releases the neighbours' flags
__device__ __forceinline__ void peer_arrive(const PeerSend &ps, int lane) {
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
        const unsigned prev = atomicAdd(&ps.hdr->arrive, 1u);
        if (prev == (unsigned)ps.n_if_chunks - 1) {
            ps.hdr->arrive = 0;
            __threadfence_system();
            const unsigned long long val = ld_volatile(&ps.hdr->halo_epoch) + 1;
            for (int k = 0; k < ps.n_nb; ++k) st_relaxed_sys(ps.flag[k], val);
        }
    }
}

struct PeerJacobiEpi {
    double omega;
    const double *__restrict__ b;
    const double *__restrict__ dinv;
    const uint8_t *__restrict__ free_m;
    const uint8_t *__restrict__ iface;
    double *__restrict__ x_out;
    double *__restrict__ s_part;
    const PeerSend *ps;
    double part[1];
    __device__ __forceinline__ void operator()(int64_t m, double s, double xo) {
        if (iface[m]) {
            s_part[m] = s;
            peer_push(*ps, (int)m, s);
            return;
        }
        double r = free_m[m] ? b[m] - s : 0.0;
        part[0] += r * r;
        if (x_out) x_out[m] = dinv ? xo + omega * (dinv[m] * r) : xo + omega * r;
    }
};

// ENERGY: part sums p_m s_m over EVERY node, the shared ones with their slab-partial s --
// i.e. the slab's element energies sum_e p_e^T A_e p_e (p = 0 at constrained nodes), whose
// sum over the ranks is p.mask(A p) without waiting for the halo (ebs_peer_matvec_sweep_put).
template <bool ENERGY = false>
struct PeerMatvecEpi {
    const uint8_t *__restrict__ free_m;
    const uint8_t *__restrict__ iface;
    double *__restrict__ q;
    const PeerSend *ps;
    double part[1];
    __device__ __forceinline__ void operator()(int64_t m, double s, double po) {
        if (iface[m]) {
            q[m] = s;  // partial; completed after the halo
            peer_push(*ps, (int)m, s);
            if (ENERGY) part[0] += po * s;
            return;
        }
        double qm = free_m[m] ? s : 0.0;
        q[m] = qm;
        part[0] += po * qm;
    }
};

// The chunk list holds the interface chunks first (clist[0, n_if_chunks)): the first
// warps of the persistent grid take them at launch, push their nodes and arrive.
template <int NB, int IDS, bool PIPE, class Epi>
__device__ __forceinline__ void peer_sweep(const SellView &v, const double *__restrict__ x,
                                           Epi &epi, const PeerSend &ps) {
    __shared__ __align__(16) int32_t stab_all[256 / LANES][SellStab<NB, IDS>::CAP];
    const int lane = threadIdx.x & (LANES - 1);
    int32_t *stab = sell_stab_init<NB, IDS>(v, stab_all);
    const XLdg xl{x};
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
    const int nwarps = (int)((gridDim.x * blockDim.x) / LANES);
    const int nlist = (int)v.nlist;
    for (int ci = warp; ci < nlist; ci += nwarps) {
        sell_chunk<NB, IDS, false, PIPE>(v, v.clist[ci], lane, stab, xl, epi);
        if (ci < ps.n_if_chunks) peer_arrive(ps, lane);
    }
}

template <int NB, int IDS>
__global__ void __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)
    k_peer_jacobi_sweep(SellView v, const double *__restrict__ x, PeerJacobiEpi epi,
                        __grid_constant__ const PeerSend ps, double *partials,
                        unsigned int *counter, double *red) {
    epi.ps = &ps;
    peer_sweep<NB, IDS, NB == 3>(v, x, epi, ps);
    double tot[1];
    if (grid_sum_last<1>(epi.part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

template <int NB, int IDS>
__global__ void __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)
    k_peer_matvec_sweep(SellView v, const double *__restrict__ p, PeerMatvecEpi<> epi,
                        __grid_constant__ const PeerSend ps, double *partials,
                        unsigned int *counter, double *red, const int32_t *stop) {
    if (stop && *stop) return;  // single-reduction PCG already stopped (ebs_dist_set_stop)
    epi.ps = &ps;
    peer_sweep<NB, IDS, false>(v, p, epi, ps);
    double tot[1];
    if (grid_sum_last<1>(epi.part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

// The slab residual r = b_p - A_p x in the rank's caller order (dist.residual_local): one
// sweep stores every node's partial residual into the caller-order r and pushes the
// interface nodes' partials to the neighbours; the combine then adds the neighbours'
// partials onto the owned shared entries.  red = 0: a plain scattered store; red = 1: the
// red.add into a -0.0-filled vector of the 1-GPU pass (operators.cu OpEpi) -- cheaper in the
// L1tex pipe for large slabs, but the fill launch costs more than that at the size of an
// 8-way C2 slab (emulated, profiles/r02_peer_scaling_c2.txt).
struct PeerResidualEpi {
    const double *__restrict__ b_int;
    const uint8_t *__restrict__ iface;
    const int32_t *__restrict__ old_of_new;
    double *__restrict__ out;
    const PeerSend *ps;
    int red;
    __device__ __forceinline__ void operator()(int64_t m, double s, double) {
        s = b_int[m] - s;
        if (red) atomicAdd(out + old_of_new[m], s);
        else out[old_of_new[m]] = s;
        if (iface[m]) peer_push(*ps, (int)m, s);
    }
};

template <int NB, int IDS>
__global__ void __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)
    k_peer_residual_sweep(SellView v, const double *__restrict__ x, PeerResidualEpi epi,
                          __grid_constant__ const PeerSend ps) {
    pdl_wait();  // PDL-launched after the x permutation
    epi.ps = &ps;
    peer_sweep<NB, IDS, false>(v, x, epi, ps);
    pdl_trigger();
}

// ------------------------------------------------------- combine + completion --
__global__ void __launch_bounds__(256)
    k_peer_combine_jacobi(__grid_constant__ const PeerRecv r, double *s, double omega,
                          const double *__restrict__ b, const double *__restrict__ dinv,
                          const uint8_t *__restrict__ free_m, const uint8_t *__restrict__ owned,
                          const double *__restrict__ x, double *__restrict__ x_out,
                          double *partials, unsigned int *counter, const double *prior,
                          double *red) {
    const unsigned long long ep = recv_wait(r);
    const int par = (int)(ep & 1);
    double part[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = r.all_if[i];
        const double acc = recv_sum(r, i, s, par);
        s[m] = acc;
        const double rr = free_m[m] ? b[m] - acc : 0.0;
        if (owned[m]) part[0] += rr * rr;
        if (x_out) x_out[m] = dinv ? x[m] + omega * (dinv[m] * rr) : x[m] + omega * rr;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0) {
        red[0] = prior ? (prior[0] + prior[1]) + tot[0] : tot[0];
        r.hdr->halo_epoch = ep + 1;
    }
}

// This rank's contribution to the fused all-reduce: dots[0..3) into slot [parity][rank] of
// every window, then the flags (one thread; the put phase of ebs_peer_allreduce).
struct RedPut {
    char *win[PEER_MAX];
    int rank, world;
};

__device__ __forceinline__ void red_put_thread(const RedPut &a, const double *dots) {
    WinHdr *h = reinterpret_cast<WinHdr *>(a.win[a.rank]);
    const unsigned long long ep = ld_volatile(&h->red_epoch);
    const int par = (int)(ep & 1);
    const double d0 = dots[0], d1 = dots[1], d2 = dots[2];
    for (int q = 0; q < a.world; ++q) {
        double *dst = win_red(a.win[q], par, a.rank);
        dst[0] = d0;
        dst[1] = d1;
        dst[2] = d2;
    }
    __threadfence_system();
    for (int q = 0; q < a.world; ++q)
        st_relaxed_sys(&reinterpret_cast<WinHdr *>(a.win[q])->red_flag[a.rank], ep + 1);
}

// One damped-Jacobi iteration k >= 1 per launch, the previous iteration's shared-node
// completion overlapped with this iteration's interior sweep (no grid barrier):
//   * the first ceil(n_if/32) warps complete iteration k-1's shared nodes (wait for the
//     neighbours' flags, rank-ordered sums, x_k there -- k_peer_combine_jacobi's work) and
//     arrive; the last one advances the halo epoch;
//   * the chunk list is [interface chunks | interior | chunks next to an interface node]:
//     interface and near-interface chunks read x_k at shared nodes, so their warps wait for
//     the arrivals (the near ones come last: by then there is nothing to wait for); the
//     interior chunks start at once -- the completion's latency hides under the interior
//     sweep.  Interface partials are pushed as in k_peer_jacobi_sweep.
// Balance: warp w sweeps the list positions w, w + nwarps, ...; when the chunk count is
// not a multiple of the warps, the warps from nlist % nwarps on have one chunk fewer, and
// the completion work and the interface chunks go to those warps (the list is read with
// the interface chunks moved to logical positions [pos0, pos0 + n_if_chunks)) -- the
// completion then costs no tail.  Waiting warps wait only for completion warps that are
// already running (resident persistent grid), never the reverse.
struct PrevJacobi {
    double *s;              // the previous sweep's own partials at the shared nodes -> totals
    const double *x_prev;   // x_{k-1}
    double *x_cur;          // x_k: the sweep's input, completed here at the shared nodes
    const uint8_t *owned;
    const double *prior;    // [previous sweep's partial, 0]
    double *red;            // ||r_{k-1}||^2 slot
    double *part_out;       // [this sweep's partial] for the next step (may alias prior[0])
    int n_near;             // near-interface chunks at the end of the list
};

__device__ __forceinline__ void wait_done_a(WinHdr *h, unsigned target) {
    if ((threadIdx.x & 31) == 0)
        while (*reinterpret_cast<volatile unsigned *>(&h->done_a) < target) __nanosleep(64);
    __syncwarp();
    __threadfence();
}

template <int NB, int IDS>
__global__ void __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)
    k_peer_jacobi_step(SellView v, PeerJacobiEpi epi, __grid_constant__ const PeerSend ps,
                       __grid_constant__ const PeerRecv pr, PrevJacobi pv, double *partials,
                       unsigned int *counter) {
    pdl_wait();  // PDL-launched after the previous iteration's step (a no-op otherwise)
    __shared__ double part_a[256];  // completion partials, parked outside the sweep's registers
    __shared__ __align__(16) int32_t stab_all[256 / LANES][SellStab<NB, IDS>::CAP];
    const int lane = threadIdx.x & (LANES - 1);
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
    const int nwarps = (int)((gridDim.x * blockDim.x) / LANES);
    const unsigned n_a = (unsigned)((pr.n_if + LANES - 1) / LANES);
    const int nlist = (int)v.nlist;
    const int n_ifc = ps.n_if_chunks;
    const int rem = nlist % nwarps;
    const int need = n_ifc > (int)n_a ? n_ifc : (int)n_a;
    // the short warps exist only when the list spans more than one round of the grid
    const int pos0 = nlist > nwarps && rem > 0 && nwarps - rem >= need ? rem : 0;
    part_a[threadIdx.x] = 0.0;
    if ((unsigned)(warp - pos0) < n_a) {  // ---- completion of iteration k-1's shared nodes ----
        const unsigned long long ep = ld_volatile(&pr.hdr->halo_epoch);
        if (lane < pr.n_src && pr.src[lane] != pr.rank)
            peer_wait(&pr.hdr->halo_flag[pr.src[lane]], ep + 1, pr.timeout_ns, &pr.hdr->error);
        __syncwarp();
        const int par = (int)(ep & 1);
        const int64_t i = (int64_t)(warp - pos0) * LANES + lane;
        if (i < pr.n_if) {
            const int64_t m = pr.all_if[i];
            const double acc = recv_sum(pr, i, pv.s, par);
            pv.s[m] = acc;
            const double rr = epi.free_m[m] ? epi.b[m] - acc : 0.0;
            if (pv.owned[m]) part_a[threadIdx.x] = rr * rr;
            pv.x_cur[m] = epi.dinv ? pv.x_prev[m] + epi.omega * (epi.dinv[m] * rr)
                                   : pv.x_prev[m] + epi.omega * rr;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            const unsigned prev = atomicAdd(&pr.hdr->arrive, 1u) + 1;  // arrive: free here
            if (prev == n_a) {
                pr.hdr->arrive = 0;
                pr.hdr->halo_epoch = ep + 1;  // every completion warp has read ep
                __threadfence();
                atomicExch(&pr.hdr->done_a, n_a);
            }
        }
    }
    // ---- the sweep of iteration k from x_k ----
    epi.ps = &ps;
    int32_t *stab = sell_stab_init<NB, IDS>(v, stab_all);
    const XLdg xl{pv.x_cur};
    const int first_near = nlist - pv.n_near;
    for (int ci = warp; ci < nlist; ci += nwarps) {
        // logical position -> list index: [pos0, pos0 + n_ifc) holds the interface chunks
        // (list[0, n_ifc)), the positions before them the list's next pos0 entries
        const bool is_if = (unsigned)(ci - pos0) < (unsigned)n_ifc;
        const int li = is_if ? ci - pos0 : (ci < pos0 ? n_ifc + ci : ci);
        if (is_if || li >= first_near) wait_done_a(pr.hdr, n_a);
        sell_chunk<NB, IDS, false, NB == 3>(v, v.clist[li], lane, stab, xl, epi);
        if (is_if) peer_arrive(ps, lane);
    }
    pdl_trigger();  // the next iteration's step may be scheduled (it waits for this grid)
    double part[2] = {part_a[threadIdx.x], epi.part[0]};
    double tot[2];
    if (grid_sum_last<2>(part, partials, counter, tot) && threadIdx.x == 0) {
        pv.red[0] = (pv.prior[0] + pv.prior[1]) + tot[0];
        pv.part_out[0] = tot[1];
        pr.hdr->done_a = 0;  // every waiter has passed
    }
}

// The single-reduction PCG's matvec sweep with the dot and the all-reduce put folded in:
// w = A u (interface partials pushed), delta = sum_e u_e^T A_e u_e over the slab's elements
// (the ENERGY epilogue: summed over the ranks it is u.mask(A u), u being 0 at constrained
// nodes), and the last block puts [gamma, delta, rr] = dots[0..3) with dots[1] := delta for
// the update kernel, which completes the shared nodes itself (ebs_peer_cg1_update_halo):
// no combine launch, and the put does not wait for the neighbours.
template <int NB, int IDS>
__global__ void __launch_bounds__(256, (NB) == 3 ? EBS_MINB2 : EBS_MINB3)
    k_peer_matvec_sweep_put(SellView v, const double *__restrict__ p, PeerMatvecEpi<true> epi,
                            __grid_constant__ const PeerSend ps, double *partials,
                            unsigned int *counter, __grid_constant__ const RedPut rp,
                            double *dots, const int32_t *stop) {
    if (stop && *stop) return;  // single-reduction PCG already stopped
    epi.ps = &ps;
    peer_sweep<NB, IDS, false>(v, p, epi, ps);
    double tot[1];
    if (grid_sum_last<1>(epi.part, partials, counter, tot) && threadIdx.x == 0) {
        dots[1] = tot[0];
        red_put_thread(rp, dots);
    }
}

__global__ void __launch_bounds__(256)
    k_peer_combine_q(__grid_constant__ const PeerRecv r, double *q,
                     const uint8_t *__restrict__ free_m, const uint8_t *__restrict__ owned,
                     const double *__restrict__ p, double *partials, unsigned int *counter,
                     const double *prior, double *red, const int32_t *stop,
                     __grid_constant__ const RedPut rp, const double *dots) {
    // a stopped single-reduction PCG: the sweep sent nothing (every rank stops at the same
    // iteration -- the decision comes from all-reduced scalars), so nothing is awaited
    if (stop && *stop) return;
    const unsigned long long ep = recv_wait(r);
    const int par = (int)(ep & 1);
    double part[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = r.all_if[i];
        const double acc = recv_sum(r, i, q, par);
        const double qm = free_m[m] ? acc : 0.0;
        q[m] = qm;
        if (owned[m]) part[0] += p[m] * qm;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0) {
        red[0] = prior ? (prior[0] + prior[1]) + tot[0] : tot[0];
        r.hdr->halo_epoch = ep + 1;
        if (dots) red_put_thread(rp, dots);
    }
}

// owned shared nodes of a caller-order residual: out[old_of_new[m]] (the own partial) +=
// the neighbours' partials in ascending rank order (the owner is the lowest touching rank)
__global__ void __launch_bounds__(256)
    k_peer_residual_combine(__grid_constant__ const PeerRecv r, const uint8_t *__restrict__ owned,
                            const int32_t *__restrict__ old_of_new, double *out,
                            unsigned int *counter) {
    pdl_wait();
    const unsigned long long ep = recv_wait(r);
    const int par = (int)(ep & 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = r.all_if[i];
        if (!owned[m]) continue;
        double acc = out[old_of_new[m]];
        for (int k = 0; k < r.n_src; ++k) {
            const int32_t q = r.pos[i * r.n_src + k];
            if (q < 0 || r.src[k] == r.rank) continue;
            acc += __ldcg(win_recv(const_cast<char *>(r.win), r.cap, r.src[k], par) + q);
        }
        out[old_of_new[m]] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        if (prev == gridDim.x - 1) {
            *counter = 0;
            r.hdr->halo_epoch = ep + 1;
        }
    }
}

// v[all_if[i]] = the rank-ordered sum (the halo of setup / residual vectors)
__global__ void __launch_bounds__(256)
    k_peer_combine(__grid_constant__ const PeerRecv r, double *v, unsigned int *counter) {
    const unsigned long long ep = recv_wait(r);
    const int par = (int)(ep & 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double acc = recv_sum(r, i, v, par);
        v[r.all_if[i]] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        if (prev == gridDim.x - 1) {
            *counter = 0;
            r.hdr->halo_epoch = ep + 1;
        }
    }
}

// v at the interface nodes into the neighbours' slots (k_peer_put over per-node entries)
__global__ void __launch_bounds__(256)
    k_peer_push_vec(__grid_constant__ const PeerSend ps, int64_t n_if,
                    const int64_t *__restrict__ all_if, const double *__restrict__ v) {
    const unsigned long long ep = ld_volatile(&ps.hdr->halo_epoch);
    const int64_t par = (int64_t)(ep & 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double val = v[all_if[i]];
        for (int e = ps.snd_off[i]; e < ps.snd_off[i + 1]; ++e)
            reinterpret_cast<double *>(ps.snd_addr[e])[par * ps.cap] = val;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&ps.hdr->arrive, 1u);
        if (prev == gridDim.x - 1) {
            ps.hdr->arrive = 0;
            __threadfence_system();
            for (int k = 0; k < ps.n_nb; ++k) st_relaxed_sys(ps.flag[k], ep + 1);
        }
    }
}

int peer_cg1_update(const RedGet &rg, const PeerRecv &hr, const uint8_t *free_m, int64_t n,
                    double *cur, const double *prev,
                    const double *rr0, double tol, int32_t *ctl, const uint8_t *owned,
                    const double *dinv, double *x, double *r, double *u, const double *w,
                    double *p, double *s, double *next, int32_t *nonfinite, void *ws,
                    void *stream);  // dist.cu

PeerSend peer_send_args(const Peer *p, int64_t n_if_chunks) {
    PeerSend ps{};
    ps.hdr = hdr_of(p);
    ps.ifx = p->ifx;
    ps.snd_off = p->snd_off;
    ps.snd_addr = p->snd_addr;
    ps.cap = p->cap;
    ps.n_if_chunks = (int)n_if_chunks;
    ps.n_nb = p->n_nb;
    for (int k = 0; k < p->n_nb; ++k)
        ps.flag[k] = &reinterpret_cast<WinHdr *>(p->win[p->nb[k]])->halo_flag[p->rank];
    return ps;
}

PeerRecv peer_recv_args(const Peer *p) {
    PeerRecv r{};
    r.hdr = hdr_of(p);
    r.win = p->win[p->rank];
    r.cap = p->cap;
    r.n_if = p->n_if;
    r.all_if = p->all_if;
    r.pos = p->pos;
    r.n_src = p->n_src;
    for (int k = 0; k < p->n_src; ++k) r.src[k] = p->src[k];
    r.rank = p->rank;
    r.timeout_ns = p->timeout_ns;
    return r;
}

struct Scratch2 {
    double *partials;
    unsigned int *counter;
};
inline Scratch2 scratch2(void *ws) {  // the layout of dist.cu's ebs_vec_workspace_bytes
    Scratch2 s;
    s.counter = reinterpret_cast<unsigned int *>(ws);
    s.partials = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + 256);
    return s;
}

// ----------------------------------------------------------------- self-test --
// The peer protocol under real concurrency on ONE GPU (the emulation the profiling guide
// prescribes: one cooperative kernel over all ranks' data, block groups as ranks), using the
// product's device functions (peer_push / peer_arrive / recv_wait / recv_sum, red_put_thread
// / red_get_block) on the ranks' real windows and halo maps.  Every iteration each rank
// pushes code(rank, global id, k) for its shared nodes and one all-reduce triple; after the
// waits it checks every shared-node sum (ascending rank order) and the reduced triple
// against the expected values.  Ranks are skewed with rank-dependent sleeps so fast ranks
// run ahead into the next epoch while slow ones still read -- any parity / epoch / fence
// error shows up as a wrong value (or a timeout).
struct StressRank {
    PeerSend ps;
    PeerRecv pr;
    RedPut rp;
    RedGet rg;
    const int64_t *gid;  // global id of each local node
    double *own;         // this rank's pushed values (the own source of recv_sum)
    int n_chunks;        // interface "chunks" of 32 shared nodes
    unsigned *bar;       // [count, generation] of the rank's block barrier
};

__device__ __forceinline__ double stress_code(int q, int64_t g, int k) {
    return (double)((int64_t)(k + 1) * 1000003 + (int64_t)q * 10007 + g);  // exact in f64
}

__device__ void rank_sync(unsigned *bar, int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == (unsigned)nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256)
    k_peer_selftest(const StressRank *__restrict__ ranks, int P, int iters,
                    unsigned long long *errors) {
    const int r = (int)((int64_t)blockIdx.x * P / gridDim.x);
    const int b0 = (int)(((int64_t)r * gridDim.x + P - 1) / P);
    const int b1 = (int)(((int64_t)(r + 1) * gridDim.x + P - 1) / P);
    const int nb = b1 - b0, bi = blockIdx.x - b0;
    const StressRank &R = ranks[r];
    const int lane = threadIdx.x & 31;
    const int warp = bi * (blockDim.x / 32) + threadIdx.x / 32, nwarps = nb * (blockDim.x / 32);
    unsigned long long bad = 0;
    for (int k = 0; k < iters; ++k) {
        if ((r + k) % 3 == 0) __nanosleep(2000 * (r + 1));  // skew the ranks
        // push: one warp per interface chunk, then the arrival that publishes the flags
        for (int c = warp; c < R.n_chunks; c += nwarps) {
            const int64_t i = (int64_t)c * 32 + lane;
            if (i < R.pr.n_if) {
                const int64_t m = R.pr.all_if[i];
                const double val = stress_code(r, R.gid[m], k);
                R.own[m] = val;
                peer_push(R.ps, (int)m, val);
            }
            peer_arrive(R.ps, lane);
        }
        rank_sync(R.bar, nb);  // the own values (other blocks of the rank) before the sums
        // combine: wait for the neighbours, check every shared node's rank-ordered sum
        const unsigned long long ep = recv_wait(R.pr);
        const int par = (int)(ep & 1);
        for (int64_t i = bi * (int64_t)blockDim.x + threadIdx.x; i < R.pr.n_if;
             i += (int64_t)nb * blockDim.x) {
            const int64_t m = R.pr.all_if[i];
            const double got = recv_sum(R.pr, i, R.own, par);
            double want = 0.0;
            for (int s = 0; s < R.pr.n_src; ++s)
                if (R.pr.pos[i * R.pr.n_src + s] >= 0) want += stress_code(R.pr.src[s], R.gid[m], k);
            if (got != want) ++bad;
        }
        rank_sync(R.bar, nb);
        const bool reduce = k % 5 == 4;  // an all-reduce syncs the ranks: only now and then,
                                         // so fast ranks can run an epoch ahead in between
        if (bi == 0 && threadIdx.x == 0) {
            R.pr.hdr->halo_epoch = ep + 1;
            if (reduce) {
                const double dots[3] = {(double)(r + 1), (double)k, (double)(2 * r)};
                red_put_thread(R.rp, dots);
            }
        }
        if (!reduce) {
            rank_sync(R.bar, nb);
            continue;
        }
        double v[3];
        const unsigned long long rep = red_get_block<3>(R.rg, v);
        if (threadIdx.x == 0) {
            const double s0 = (double)P * (P + 1) / 2, s2 = (double)P * (P - 1);
            if (v[0] != s0 || v[1] != (double)k * P || v[2] != s2) ++bad;
        }
        rank_sync(R.bar, nb);
        if (bi == 0 && threadIdx.x == 0)
            reinterpret_cast<WinHdr *>(R.rg.win)->red_epoch = rep + 1;
        rank_sync(R.bar, nb);
    }
    if (bad) atomicAdd(errors, bad);
}

}  // namespace ebs

using namespace ebs;

extern "C" {

size_t ebs_peer_window_bytes(int64_t cap) { return window_bytes(cap < 0 ? 0 : cap); }

int ebs_peer_window_alloc(int64_t cap, void **win, void *handle_out) {
    EBS_TRY
    EBS_REQUIRE(cap >= 0 && win, "bad arguments");
    void *p = nullptr;
    CU(cudaMalloc(&p, window_bytes(cap)));
    cudaError_t e = cudaMemset(p, 0, window_bytes(cap));
    if (e == cudaSuccess && handle_out) {
        cudaIpcMemHandle_t h;
        e = cudaIpcGetMemHandle(&h, p);
        if (e == cudaSuccess) std::memcpy(handle_out, &h, sizeof h);
    }
    if (e != cudaSuccess) {
        cudaFree(p);
        CU(e);
    }
    CU(cudaDeviceSynchronize());
    *win = p;
    EBS_CATCH
}

int ebs_peer_window_open(const void *handle, void **win) {
    EBS_TRY
    EBS_REQUIRE(handle && win, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void *p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();  // not sticky: clear it, so the next launch check does not see it
        CU(e);
    }
    *win = p;
    EBS_CATCH
}

int ebs_peer_window_close(void *win) {
    EBS_TRY
    if (win) CU(cudaIpcCloseMemHandle(win));
    EBS_CATCH
}

int ebs_peer_window_free(void *win) {
    EBS_TRY
    if (win) CU(cudaFree(win));
    EBS_CATCH
}

int ebs_peer_create(int rank, int world, int64_t cap, void *const *wins, double timeout_s,
                    ebs_peer_t *out) {
    EBS_TRY
    EBS_REQUIRE(world >= 1 && world <= PEER_MAX && rank >= 0 && rank < world && cap >= 0 &&
                    wins && out,
                "bad arguments (1 <= world <= %d)", PEER_MAX);
    for (int q = 0; q < world; ++q) EBS_REQUIRE(wins[q], "null window of rank %d", q);
    Peer *p = new Peer();
    p->rank = rank;
    p->world = world;
    p->cap = cap;
    p->timeout_ns = timeout_s < 0 ? (long long)4e18 : (long long)(timeout_s * 1e9);
    for (int q = 0; q < world; ++q) p->win[q] = static_cast<char *>(wins[q]);
    p->n_src = 1;
    p->src[0] = rank;
    *out = reinterpret_cast<ebs_peer_t>(p);
    EBS_CATCH
}

static void peer_clear_halo(Peer *p) {
    dfree(p->all_if);
    dfree(p->ifx);
    dfree(p->snd_off);
    dfree(p->snd_addr);
    dfree(p->pos);
    p->n_nb = 0;
    p->n_if = 0;
    p->n_src = 1;
    p->src[0] = p->rank;
}

int ebs_peer_destroy(ebs_peer_t peer) {
    EBS_TRY
    if (!peer) return EBS_OK;
    Peer *p = reinterpret_cast<Peer *>(peer);
    peer_clear_halo(p);
    delete p;
    EBS_CATCH
}

int ebs_peer_set_halo(ebs_peer_t peer, int64_t n_local, int n_nb, const int32_t *nb_ranks,
                      const int64_t *nb_len, const int64_t *const *nb_idx, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && n_local >= 0 && n_nb >= 0 && (n_nb == 0 || (nb_ranks && nb_len && nb_idx)),
                "bad arguments");
    Peer *p = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(n_nb < p->world, "more neighbours than ranks");
    cudaStream_t s = S(stream);
    std::vector<std::vector<int64_t>> idx(n_nb);
    for (int k = 0; k < n_nb; ++k) {
        EBS_REQUIRE(nb_ranks[k] >= 0 && nb_ranks[k] < p->world && nb_ranks[k] != p->rank &&
                        (k == 0 || nb_ranks[k] > nb_ranks[k - 1]),
                    "neighbour ranks must be ascending, distinct from the caller");
        EBS_REQUIRE(nb_len[k] >= 0 && nb_len[k] <= p->cap, "interface %d longer than the window "
                    "capacity (%lld > %lld)", k, (long long)nb_len[k], (long long)p->cap);
        idx[k].resize(nb_len[k]);
        if (nb_len[k])
            CU(cudaMemcpyAsync(idx[k].data(), nb_idx[k], sizeof(int64_t) * nb_len[k],
                               cudaMemcpyDeviceToHost, s));
    }
    CU(cudaStreamSynchronize(s));
    std::vector<int64_t> all;
    for (int k = 0; k < n_nb; ++k) {
        for (int64_t m : idx[k]) EBS_REQUIRE(m >= 0 && m < n_local, "interface node out of range");
        all.insert(all.end(), idx[k].begin(), idx[k].end());
    }
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    const int64_t n_if = (int64_t)all.size();
    EBS_REQUIRE(n_local < (1ll << 31) && n_if < (1ll << 31), "slab too large");
    std::vector<int32_t> ifx(n_local, -1);
    for (int64_t i = 0; i < n_if; ++i) ifx[all[i]] = (int32_t)i;
    // send entries per interface node (neighbours ascending) and the combine positions
    std::vector<std::vector<std::pair<int, int64_t>>> ent(n_if);
    for (int k = 0; k < n_nb; ++k)
        for (int64_t j = 0; j < nb_len[k]; ++j) ent[ifx[idx[k][j]]].push_back({k, j});
    std::vector<int32_t> off(n_if + 1, 0);
    std::vector<unsigned long long> addr;
    int srcs[PEER_MAX];
    int n_src = 0;
    {
        std::vector<int> r(nb_ranks, nb_ranks + n_nb);
        r.push_back(p->rank);
        std::sort(r.begin(), r.end());
        for (int v : r) srcs[n_src++] = v;
    }
    std::vector<int32_t> pos((size_t)n_if * n_src, -1);
    for (int64_t i = 0; i < n_if; ++i) {
        off[i + 1] = off[i] + (int32_t)ent[i].size();
        for (auto &e : ent[i]) {
            const int q = nb_ranks[e.first];
            addr.push_back(reinterpret_cast<unsigned long long>(
                win_recv(p->win[q], p->cap, p->rank, 0) + e.second));
            const int ks = (int)(std::find(srcs, srcs + n_src, q) - srcs);
            pos[(size_t)i * n_src + ks] = (int32_t)e.second;
        }
        const int self = (int)(std::find(srcs, srcs + n_src, p->rank) - srcs);
        pos[(size_t)i * n_src + self] = (int32_t)all[i];
    }
    peer_clear_halo(p);
    p->n_local = n_local;
    p->n_nb = n_nb;
    for (int k = 0; k < n_nb; ++k) {
        p->nb[k] = nb_ranks[k];
        p->len[k] = nb_len[k];
    }
    p->n_if = n_if;
    p->n_src = n_src;
    for (int k = 0; k < n_src; ++k) p->src[k] = srcs[k];
    p->all_if = dmalloc<int64_t>(n_if);
    p->ifx = dmalloc<int32_t>(n_local);
    p->snd_off = dmalloc<int32_t>(n_if + 1);
    p->snd_addr = dmalloc<unsigned long long>(addr.size());
    p->pos = dmalloc<int32_t>(pos.size());
    if (n_if) CU(cudaMemcpyAsync(p->all_if, all.data(), sizeof(int64_t) * n_if, cudaMemcpyHostToDevice, s));
    if (n_local) CU(cudaMemcpyAsync(p->ifx, ifx.data(), sizeof(int32_t) * n_local, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(p->snd_off, off.data(), sizeof(int32_t) * (n_if + 1), cudaMemcpyHostToDevice, s));
    if (!addr.empty())
        CU(cudaMemcpyAsync(p->snd_addr, addr.data(), sizeof(unsigned long long) * addr.size(),
                           cudaMemcpyHostToDevice, s));
    if (!pos.empty())
        CU(cudaMemcpyAsync(p->pos, pos.data(), sizeof(int32_t) * pos.size(), cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));  // host vectors go out of scope
    EBS_CATCH
}

int ebs_peer_status(ebs_peer_t peer, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    unsigned int err = 0;
    CU(cudaMemcpyAsync(&err, &hdr_of(p)->error, sizeof err, cudaMemcpyDeviceToHost, S(stream)));
    CU(cudaStreamSynchronize(S(stream)));
    if (err) {
        set_error("peer exchange timed out waiting for another rank (rank %d of %d)", p->rank,
                  p->world);
        return EBS_ENCCL;
    }
    EBS_CATCH
}

int ebs_peer_allreduce(ebs_peer_t peer, double *buf, int64_t n, int mode, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && (buf || n == 0) && n >= 0 && mode >= 0 && mode <= 2, "bad arguments");
    Peer *p = reinterpret_cast<Peer *>(peer);
    RedArgs a{};
    for (int q = 0; q < p->world; ++q) a.win[q] = p->win[q];
    a.rank = p->rank;
    a.world = p->world;
    a.timeout_ns = p->timeout_ns;
    EBS_REQUIRE(mode == 0 || n <= PEER_RED_MAX, "split all-reduce phases take <= %d values",
                PEER_RED_MAX);
    for (int64_t o = 0; o < n; o += PEER_RED_MAX) {
        a.n = (int)std::min<int64_t>(PEER_RED_MAX, n - o);
        k_peer_allreduce<<<1, 256, 0, S(stream)>>>(a, buf + o, mode);
        LAUNCHED();
    }
    EBS_CATCH
}

int ebs_peer_send(ebs_peer_t peer, const double *const *bufs, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->n_nb == 0 || bufs, "null buffers");
    PutArgs a{};
    a.hdr = hdr_of(p);
    a.n_nb = p->n_nb;
    a.cap = p->cap;
    a.off[0] = 0;
    for (int k = 0; k < p->n_nb; ++k) {
        EBS_REQUIRE(bufs[k] || p->len[k] == 0, "null buffer %d", k);
        a.src[k] = bufs[k];
        a.dst[k] = win_recv(p->win[p->nb[k]], p->cap, p->rank, 0);
        a.flag[k] = &reinterpret_cast<WinHdr *>(p->win[p->nb[k]])->halo_flag[p->rank];
        a.off[k + 1] = a.off[k] + p->len[k];
    }
    k_peer_put<<<grid_for(a.off[p->n_nb], 256, sm_count()), 256, 0, S(stream)>>>(a);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_recv(ebs_peer_t peer, double *const *out, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && ws, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->n_nb == 0 || out, "null outputs");
    GetArgs a{};
    a.hdr = hdr_of(p);
    a.n_nb = p->n_nb;
    a.cap = p->cap;
    a.timeout_ns = p->timeout_ns;
    a.off[0] = 0;
    for (int k = 0; k < p->n_nb; ++k) {
        EBS_REQUIRE(out[k] || p->len[k] == 0, "null output %d", k);
        a.nb[k] = p->nb[k];
        a.slot[k] = win_recv(p->win[p->rank], p->cap, p->nb[k], 0);
        a.out[k] = out[k];
        a.off[k + 1] = a.off[k] + p->len[k];
    }
    k_peer_get<<<grid_for(a.off[p->n_nb], 256, sm_count()), 256, 0, S(stream)>>>(
        a, scratch2(ws).counter);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_push(ebs_peer_t peer, const double *v, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && v, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    const PeerSend ps = peer_send_args(p, 0);
    k_peer_push_vec<<<grid_for(p->n_if, 256, sm_count()), 256, 0, S(stream)>>>(ps, p->n_if,
                                                                               p->all_if, v);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_combine(ebs_peer_t peer, double *v, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && v && ws, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    const PeerRecv r = peer_recv_args(p);
    k_peer_combine<<<grid_for(p->n_if, 256, sm_count()), 256, 0, S(stream)>>>(
        r, v, scratch2(ws).counter);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_jacobi_sweep(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks, int64_t n_list,
                          int64_t n_if_chunks, double omega, const double *x, double *x_out,
                          const double *b, const double *dinv, const uint8_t *iface,
                          double *s_part, double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && peer && x && b && iface && s_part && red && ws, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Peer *pr = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(n_list >= 1 && chunks && n_if_chunks >= 0 && n_if_chunks <= n_list,
                "bad chunk list");
    EBS_REQUIRE(pr->n_local == p->n_n, "peer halo set for %lld nodes, plan has %lld",
                (long long)pr->n_local, (long long)p->n_n);
    EBS_REQUIRE((n_if_chunks > 0) == (pr->n_nb > 0), "interface chunks without neighbours "
                "(or the reverse)");
    const Scratch2 sc = scratch2(ws);
    const PeerSend ps = peer_send_args(pr, n_if_chunks);
    PeerJacobiEpi epi{omega, b, dinv, p->free_int, iface, x_out, s_part, nullptr, {0.0}};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_PJ(NB_, IDS_)                                                                  \
    {                                                                                      \
        auto kern = k_peer_jacobi_sweep<NB_, IDS_>;                                        \
        const int grid = persistent_grid((const void *)kern, 256,                          \
                                         (n_list * LANES + 255) / 256, 0);                 \
        kern<<<grid, 256, 0, S(stream)>>>(v, x, epi, ps, sc.partials, sc.counter, red);    \
    }
    EBS_SELL_DISPATCH(p, EBS_PJ);
#undef EBS_PJ
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_matvec_sweep(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks, int64_t n_list,
                          int64_t n_if_chunks, const double *pv, double *q, const uint8_t *iface,
                          double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && peer && pv && q && iface && red && ws, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Peer *pr = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(n_list >= 1 && chunks && n_if_chunks >= 0 && n_if_chunks <= n_list,
                "bad chunk list");
    EBS_REQUIRE(pr->n_local == p->n_n, "peer halo set for %lld nodes, plan has %lld",
                (long long)pr->n_local, (long long)p->n_n);
    EBS_REQUIRE((n_if_chunks > 0) == (pr->n_nb > 0), "interface chunks without neighbours "
                "(or the reverse)");
    const Scratch2 sc = scratch2(ws);
    const PeerSend ps = peer_send_args(pr, n_if_chunks);
    PeerMatvecEpi<> epi{p->free_int, iface, q, nullptr, {0.0}};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_PM(NB_, IDS_)                                                                  \
    {                                                                                      \
        auto kern = k_peer_matvec_sweep<NB_, IDS_>;                                        \
        const int grid = persistent_grid((const void *)kern, 256,                          \
                                         (n_list * LANES + 255) / 256, 0);                 \
        kern<<<grid, 256, 0, S(stream)>>>(v, pv, epi, ps, sc.partials, sc.counter, red,    \
                                          p->dist_stop);                                   \
    }
    EBS_SELL_DISPATCH(p, EBS_PM);
#undef EBS_PM
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_combine_jacobi(ebs_peer_t peer, double *s, double omega, const double *b,
                            const double *dinv, const uint8_t *free_m, const uint8_t *owned,
                            const double *x, double *x_out, const double *prior, double *red,
                            void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && s && b && free_m && owned && x && red && ws, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    const Scratch2 sc = scratch2(ws);
    const PeerRecv r = peer_recv_args(p);
    const int grid = persistent_grid((const void *)k_peer_combine_jacobi, 256,
                                     (p->n_if + 255) / 256, 0);
    k_peer_combine_jacobi<<<grid, 256, 0, S(stream)>>>(r, s, omega, b, dinv, free_m, owned, x,
                                                       x_out, sc.partials, sc.counter, prior, red);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_combine_q(ebs_peer_t peer, double *q, const uint8_t *free_m, const uint8_t *owned,
                       const double *pv, const double *prior, double *red, const int32_t *stop,
                       const double *dots, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && q && free_m && owned && pv && red && ws, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    const Scratch2 sc = scratch2(ws);
    const PeerRecv r = peer_recv_args(p);
    const int grid = persistent_grid((const void *)k_peer_combine_q, 256, (p->n_if + 255) / 256, 0);
    RedPut rp{};
    for (int k = 0; k < p->world; ++k) rp.win[k] = p->win[k];
    rp.rank = p->rank;
    rp.world = p->world;
    k_peer_combine_q<<<grid, 256, 0, S(stream)>>>(r, q, free_m, owned, pv, sc.partials,
                                                  sc.counter, prior, red, stop, rp, dots);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_residual_sweep(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks,
                            int64_t n_list, int64_t n_if_chunks, const double *x_int, double *out,
                            const int32_t *out_map, const uint8_t *iface, int flags,
                            void *stream) {
    EBS_TRY
    EBS_REQUIRE(flags == 0 || flags == EBS_APPLY_ADD, "bad flags %d", flags);
    EBS_REQUIRE(plan && peer && x_int && out && out_map && iface, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Peer *pr = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->has_A && p->has_be, "residual needs an operator loaded with b_e");
    EBS_REQUIRE(n_list >= 1 && chunks && n_if_chunks >= 0 && n_if_chunks <= n_list,
                "bad chunk list");
    EBS_REQUIRE(pr->n_local == p->n_n, "peer halo set for %lld nodes, plan has %lld",
                (long long)pr->n_local, (long long)p->n_n);
    EBS_REQUIRE((n_if_chunks > 0) == (pr->n_nb > 0), "interface chunks without neighbours "
                "(or the reverse)");
    const PeerSend ps = peer_send_args(pr, n_if_chunks);
    PeerResidualEpi epi{p->b_int, iface, out_map, out, nullptr, flags == EBS_APPLY_ADD ? 1 : 0};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_PR(NB_, IDS_)                                                                  \
    {                                                                                      \
        auto kern = k_peer_residual_sweep<NB_, IDS_>;                                      \
        const int grid = persistent_grid((const void *)kern, 256,                          \
                                         (n_list * LANES + 255) / 256, 0);                 \
        launch_pdl(kern, grid, 256, 0, S(stream), v, x_int, epi, ps);                      \
    }
    EBS_SELL_DISPATCH(p, EBS_PR);
#undef EBS_PR
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_residual_combine(ebs_peer_t peer, const uint8_t *owned, const int32_t *out_map,
                              double *out, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && owned && out_map && out && ws, "null argument");
    Peer *p = reinterpret_cast<Peer *>(peer);
    const PeerRecv r = peer_recv_args(p);
    launch_pdl(k_peer_residual_combine, grid_for(p->n_if, 256, sm_count()), 256, 0, S(stream),
               r, owned, out_map, out, scratch2(ws).counter);
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_selftest(ebs_peer_t const *peers, const int64_t *const *global_ids, int P,
                      int iters, int64_t *n_errors, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peers && global_ids && n_errors && P >= 1 && P <= PEER_MAX && iters >= 0,
                "bad arguments");
    cudaStream_t s = S(stream);
    std::vector<StressRank> h(P);
    std::vector<double *> owns(P, nullptr);
    unsigned *bars = dmalloc<unsigned>(2 * P);
    unsigned long long *err = dmalloc<unsigned long long>(1);
    StressRank *d = dmalloc<StressRank>(P);
    CU(cudaMemsetAsync(bars, 0, sizeof(unsigned) * 2 * P, s));
    CU(cudaMemsetAsync(err, 0, sizeof(unsigned long long), s));
    for (int r = 0; r < P; ++r) {
        const Peer *p = reinterpret_cast<const Peer *>(peers[r]);
        EBS_REQUIRE(p && p->rank == r && p->world == P && global_ids[r], "peer %d", r);
        const int nc = (int)((p->n_if + 31) / 32);
        h[r].ps = peer_send_args(p, nc);
        h[r].pr = peer_recv_args(p);
        for (int q = 0; q < P; ++q) h[r].rp.win[q] = p->win[q];
        h[r].rp.rank = r;
        h[r].rp.world = P;
        h[r].rg = RedGet{p->win[r], P, p->timeout_ns};
        h[r].gid = global_ids[r];
        owns[r] = dmalloc<double>(p->n_local);
        h[r].own = owns[r];
        h[r].n_chunks = nc;
        h[r].bar = bars + 2 * r;
        EBS_REQUIRE((nc > 0) == (p->n_nb > 0), "peer %d: interface without neighbours", r);
    }
    CU(cudaMemcpyAsync(d, h.data(), sizeof(StressRank) * P, cudaMemcpyHostToDevice, s));
    int per_sm = 0, sms = 0, dev = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peer_selftest, 256, 0));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::min(per_sm * sms, 16 * P);  // co-resident: ranks spin on each other
    void *args[] = {(void *)&d, (void *)&P, (void *)&iters, (void *)&err};
    CU(cudaLaunchCooperativeKernel((const void *)k_peer_selftest, dim3(grid), dim3(256), args, 0, s));
    LAUNCHED();
    unsigned long long e = 0;
    CU(cudaMemcpyAsync(&e, err, sizeof e, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *n_errors = (int64_t)e;
    for (double *o : owns) cudaFree(o);
    cudaFree(bars);
    cudaFree(err);
    cudaFree(d);
    EBS_CATCH
}

int ebs_peer_jacobi_step(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks, int64_t n_list,
                         int64_t n_if_chunks, int64_t n_near, double omega, const double *x_prev,
                         double *x_cur, double *x_out, const double *b, const double *dinv,
                         const uint8_t *iface, const uint8_t *owned, double *s_part,
                         const double *prior, double *red_prev, double *part_out, void *ws,
                         void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && peer && x_prev && x_cur && b && iface && owned && s_part && prior &&
                    red_prev && part_out && ws,
                "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Peer *pr = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(n_list >= 1 && chunks && n_if_chunks >= 0 && n_near >= 0 &&
                    n_if_chunks + n_near <= n_list,
                "bad chunk list");
    EBS_REQUIRE(pr->n_local == p->n_n, "peer halo set for %lld nodes, plan has %lld",
                (long long)pr->n_local, (long long)p->n_n);
    EBS_REQUIRE((n_if_chunks > 0) == (pr->n_nb > 0), "interface chunks without neighbours "
                "(or the reverse)");
    const Scratch2 sc = scratch2(ws);
    const PeerSend ps = peer_send_args(pr, n_if_chunks);
    const PeerRecv rv = peer_recv_args(pr);
    PeerJacobiEpi epi{omega, b, dinv, p->free_int, iface, x_out, s_part, nullptr, {0.0}};
    PrevJacobi pv{s_part, x_prev, x_cur, owned, prior, red_prev, part_out, (int)n_near};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_PS(NB_, IDS_)                                                                  \
    {                                                                                      \
        auto kern = k_peer_jacobi_step<NB_, IDS_>;                                         \
        const int grid = persistent_grid((const void *)kern, 256,                          \
                                         (n_list * LANES + 255) / 256, 0);                 \
        EBS_REQUIRE((int64_t)grid * 8 >= (rv.n_if + LANES - 1) / LANES,                    \
                    "more shared nodes than the grid's completion warps");                 \
        launch_pdl(kern, grid, 256, 0, S(stream), v, epi, ps, rv, pv, sc.partials,         \
                   sc.counter);                                                            \
    }
    EBS_SELL_DISPATCH(p, EBS_PS);
#undef EBS_PS
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_matvec_sweep_put(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks,
                              int64_t n_list, int64_t n_if_chunks, const double *pv, double *q,
                              const uint8_t *iface, double *dots, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && peer && pv && q && iface && dots && ws, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    Peer *pr = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(n_list >= 1 && chunks && n_if_chunks >= 0 && n_if_chunks <= n_list,
                "bad chunk list");
    EBS_REQUIRE(pr->n_local == p->n_n, "peer halo set for %lld nodes, plan has %lld",
                (long long)pr->n_local, (long long)p->n_n);
    EBS_REQUIRE((n_if_chunks > 0) == (pr->n_nb > 0), "interface chunks without neighbours "
                "(or the reverse)");
    const Scratch2 sc = scratch2(ws);
    const PeerSend ps = peer_send_args(pr, n_if_chunks);
    RedPut rp{};
    for (int k = 0; k < pr->world; ++k) rp.win[k] = pr->win[k];
    rp.rank = pr->rank;
    rp.world = pr->world;
    PeerMatvecEpi<true> epi{p->free_int, iface, q, nullptr, {0.0}};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_PMP(NB_, IDS_)                                                                 \
    {                                                                                      \
        auto kern = k_peer_matvec_sweep_put<NB_, IDS_>;                                    \
        const int grid = persistent_grid((const void *)kern, 256,                          \
                                         (n_list * LANES + 255) / 256, 0);                 \
        kern<<<grid, 256, 0, S(stream)>>>(v, pv, epi, ps, sc.partials, sc.counter, rp,     \
                                          dots, p->dist_stop);                             \
    }
    EBS_SELL_DISPATCH(p, EBS_PMP);
#undef EBS_PMP
    LAUNCHED();
    EBS_CATCH
}

int ebs_peer_cg1_update(ebs_peer_t peer, int64_t n, double *cur, const double *prev,
                        const double *rr0, double tol, int32_t *ctl, const uint8_t *owned,
                        const double *dinv, double *x, double *r, double *u, const double *w,
                        double *p, double *s, double *next, int32_t *nonfinite, void *ws,
                        void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer, "null argument");
    Peer *pr = reinterpret_cast<Peer *>(peer);
    const RedGet rg{pr->win[pr->rank], pr->world, pr->timeout_ns};
    return peer_cg1_update(rg, PeerRecv{}, nullptr, n, cur, prev, rr0, tol, ctl, owned, dinv, x,
                           r, u, w, p, s, next, nonfinite, ws, stream);
    EBS_CATCH
}

int ebs_peer_cg1_update_halo(ebs_peer_t peer, int64_t n, double *cur, const double *prev,
                             const double *rr0, double tol, int32_t *ctl, const uint8_t *owned,
                             const uint8_t *free_m, const double *dinv, double *x, double *r,
                             double *u, double *w, double *p, double *s, double *next,
                             int32_t *nonfinite, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(peer && free_m && w, "null argument");
    Peer *pr = reinterpret_cast<Peer *>(peer);
    EBS_REQUIRE(pr->n_local == n, "peer halo set for %lld nodes, vectors have %lld",
                (long long)pr->n_local, (long long)n);
    const RedGet rg{pr->win[pr->rank], pr->world, pr->timeout_ns};
    const PeerRecv hr = peer_recv_args(pr);
    return peer_cg1_update(rg, hr, free_m, n, cur, prev, rr0, tol, ctl, owned, dinv, x, r, u, w,
                           p, s, next, nonfinite, ws, stream);
    EBS_CATCH
}

}  // extern "C"

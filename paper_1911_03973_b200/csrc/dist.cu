// dist.cu -- vector kernels of the element-slab multi-GPU path.
//
// A rank owns the elements [lo, hi) of np.linspace(0, n_e, P+1) (operators.py:100) and a
// plan over the nodes they touch.  Its SELL pass yields partial node sums; interface
// partials are exchanged with the slab neighbours by the host (NCCL P2P) and combined in
// ascending rank order with ebs_index_fill / ebs_scatter_add / ebs_index_copy, so every
// rank holds identical values on shared nodes.  Dots and norms sum OWNED nodes only
// (owner = lowest rank touching the node) and are then all-reduced.  All reductions here
// are fixed-order (deterministic for a fixed launch configuration).
#include "ebs_internal.cuh"
#include "peer.cuh"

namespace ebs {

__global__ void k_index_fill(int64_t n, const int64_t *__restrict__ idx, double value,
                             double *__restrict__ v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[idx[i]] = value;
}

__global__ void k_index_copy(int64_t n, const int64_t *__restrict__ idx,
                             const double *__restrict__ src, double *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[idx[i]] = src[idx[i]];
}

// dst[dst_idx[i]] = src[src_idx[i]]  (owned results back to the caller's numbering)
__global__ void k_index_move(int64_t n, const int64_t *__restrict__ src_idx,
                             const double *__restrict__ src, const int64_t *__restrict__ dst_idx,
                             double *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[dst_idx[i]] = src[src_idx[i]];
}

// dst[dst_idx[i]] += src[src_idx[i]]  (neighbour partials onto an owned entry)
__global__ void k_index_add(int64_t n, const int64_t *__restrict__ src_idx,
                            const double *__restrict__ src, const int64_t *__restrict__ dst_idx,
                            double *__restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[dst_idx[i]] += src[src_idx[i]];
}

// r = free ? b - s : 0;  x_out = x + omega*(dinv*r) (or x + omega*r);  red[0] = sum_owned r^2
__global__ void __launch_bounds__(256)
    k_vec_jacobi(int64_t n, double omega, const double *__restrict__ b,
                 const double *__restrict__ s, const double *__restrict__ dinv,
                 const uint8_t *__restrict__ free_m, const uint8_t *__restrict__ owned,
                 const double *__restrict__ x, double *__restrict__ x_out,
                 double *__restrict__ r_out, double *partials, unsigned int *counter,
                 double *red, int32_t *nonfinite) {
    double part[1] = {0.0};
    bool bad = false;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        double r = free_m[m] ? b[m] - s[m] : 0.0;
        if (owned[m]) part[0] += r * r;
        if (r_out) r_out[m] = r;
        if (x_out) {
            double xn = dinv ? x[m] + omega * (dinv[m] * r) : x[m] + omega * r;
            x_out[m] = xn;
            bad |= !isfinite(xn);
        }
    }
    if (bad) atomicOr(nonfinite, 1);
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

// q = free ? q : 0;  red[0] = sum_owned p*q
__global__ void __launch_bounds__(256)
    k_vec_pcg_q(int64_t n, const uint8_t *__restrict__ free_m, const uint8_t *__restrict__ owned,
                const double *__restrict__ p, double *__restrict__ q, double *partials,
                unsigned int *counter, double *red) {
    double part[1] = {0.0};
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        double qm = free_m[m] ? q[m] : 0.0;
        q[m] = qm;
        if (owned[m]) part[0] += p[m] * qm;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

// alpha = pq != 0 ? rz/pq : 0 (device scalars rz, pq);  x += alpha p;  r -= alpha q;
// red = [sum_owned r^2, sum_owned r*(dinv*r)]
// ILP-4: four independent node updates in flight per thread (the nodes a thread visits,
// and the order it sums them in, are those of the plain grid-stride loop)
constexpr int VEC_ILP = 4;

__global__ void __launch_bounds__(256)
    k_vec_pcg_update(int64_t n, const double *__restrict__ rz_p, const double *__restrict__ pq_p,
                     const uint8_t *__restrict__ owned, const double *__restrict__ dinv,
                     double *__restrict__ x, double *__restrict__ r, const double *__restrict__ p,
                     const double *__restrict__ q, double *partials, unsigned int *counter,
                     double *red, int32_t *nonfinite) {
    const double rz = rz_p[0], pq = pq_p[0];
    const double alpha = pq != 0.0 ? rz / pq : 0.0;
    double part[2] = {0.0, 0.0};
    bool bad = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n;
         base += stride * VEC_ILP) {
        double xv[VEC_ILP], rv[VEC_ILP], pv[VEC_ILP], qv[VEC_ILP], dv[VEC_ILP];
        uint8_t ow[VEC_ILP];
#pragma unroll
        for (int u = 0; u < VEC_ILP; ++u) {
            const int64_t m = base + u * stride;
            const bool ok = m < n;
            xv[u] = ok ? x[m] : 0.0;
            rv[u] = ok ? r[m] : 0.0;
            pv[u] = ok ? p[m] : 0.0;
            qv[u] = ok ? q[m] : 0.0;
            ow[u] = ok ? owned[m] : 0;
            dv[u] = ok ? dinv[m] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < VEC_ILP; ++u) {
            const int64_t m = base + u * stride;
            if (m < n) {
                const double xn = xv[u] + alpha * pv[u];
                const double rn = rv[u] - alpha * qv[u];
                x[m] = xn;
                r[m] = rn;
                bad |= !isfinite(xn);
                if (ow[u]) {
                    part[0] += rn * rn;
                    part[1] += rn * (dv[u] * rn);
                }
            }
        }
    }
    if (bad) atomicOr(nonfinite, 1);
    double tot[2];
    if (grid_sum_last<2>(part, partials, counter, tot) && threadIdx.x == 0) {
        red[0] = tot[0];
        red[1] = tot[1];
    }
}

// beta = rz_old != 0 ? rz_new/rz_old : 0;  p = dinv*r + beta*p
__global__ void __launch_bounds__(256)
    k_vec_pcg_direction(int64_t n, const double *__restrict__ rz_old,
                        const double *__restrict__ rz_new, const double *__restrict__ dinv,
                        const double *__restrict__ r, double *__restrict__ p) {
    const double beta = rz_old[0] != 0.0 ? rz_new[0] / rz_old[0] : 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n;
         base += stride * VEC_ILP) {
        double rv[VEC_ILP], pv[VEC_ILP], dv[VEC_ILP];
#pragma unroll
        for (int u = 0; u < VEC_ILP; ++u) {
            const int64_t m = base + u * stride;
            const bool ok = m < n;
            rv[u] = ok ? r[m] : 0.0;
            pv[u] = ok ? p[m] : 0.0;
            dv[u] = ok ? dinv[m] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < VEC_ILP; ++u) {
            const int64_t m = base + u * stride;
            if (m < n) p[m] = dv[u] * rv[u] + beta * pv[u];
        }
    }
}

// Single-reduction Jacobi-PCG (Chronopoulos-Gear): the three dots of an iteration,
// [gamma = r.u, delta = w.u, rr = r.r], are all-reduced together (one collective per
// iteration instead of two).  cur = those of iteration k (+ cur[3] = alpha_k, written here),
// prev = iteration k-1 (prev[0] == 0: first iteration, beta = 0):
//   beta = gamma_k / gamma_{k-1};  alpha = gamma_k / (delta_k - beta gamma_k / alpha_{k-1})
//   p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s;  u = dinv r
//   next = [sum_owned r.u, (delta: the matvec), sum_owned r.r]
// ctl = [stop, k_stop, k, diverged]: the loop rules of _iterate (solvers.py:117-160) on the
// device -- stop when ||r_k|| <= tol ||r_0|| (tol >= 0) or ||r_k|| is not finite; every
// later launch (and the plan's fused matvec sweeps, ebs_dist_set_stop) is a no-op.
// rg.win != nullptr (ebs_peer_cg1_update): cur[0..2] are not reduced yet -- every block
// waits for the ranks' contributions in the peer window (put by ebs_peer_combine_q) and adds
// them in rank order; block 0 stores the sums in cur, the last block advances the window's
// all-reduce epoch (also on the stopping launch, so every rank's epoch stays in step).
#ifndef EBS_CG1_MINB
#define EBS_CG1_MINB 1
#endif
__global__ void __launch_bounds__(256, EBS_CG1_MINB)
    k_vec_cg1_update(int64_t n, double *cur, const double *__restrict__ prev,
                     double *rr0, double tol, int32_t *ctl,
                     const uint8_t *__restrict__ owned, const double *__restrict__ dinv,
                     double *__restrict__ x, double *__restrict__ r, double *__restrict__ u,
                     double *w, double *__restrict__ p,
                     double *__restrict__ s, double *partials, unsigned int *counter,
                     double *next, int32_t *nonfinite, const RedGet rg,
                     const PeerRecv hr, const uint8_t *__restrict__ free_m) {
    if (ctl && ctl[0]) return;
    if (hr.hdr) {
        // the previous sweep's shared nodes of w (ebs_peer_matvec_sweep_put pushed the
        // partials and put the dots without waiting): rank-ordered sums, masked, then a grid
        // barrier so every thread sees the completed w
        const unsigned long long hep = recv_wait(hr);
        const int hpar = (int)(hep & 1);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hr.n_if;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t m = hr.all_if[i];
            const double acc = recv_sum(hr, i, w, hpar);
            w[m] = free_m[m] ? acc : 0.0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned arrived = atomicAdd(&hr.hdr->done_a, 1u) + 1;
            if (arrived == gridDim.x) {  // every block has read hep and finished its nodes
                hr.hdr->halo_epoch = hep + 1;
                __threadfence();
                atomicAdd(&hr.hdr->done_a, 1u);
            }
            while (*reinterpret_cast<volatile unsigned *>(&hr.hdr->done_a) < gridDim.x + 1)
                __nanosleep(64);
            __threadfence();
        }
        __syncthreads();
    }
    double gamma, delta, rr;
    unsigned long long ep = 0;
    if (rg.win) {
        double v[3];
        ep = red_get_block<3>(rg, v);
        gamma = v[0];
        delta = v[1];
        rr = v[2];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            cur[0] = gamma;
            cur[1] = delta;
            cur[2] = rr;
            cur[4] = rr;  // history copy: [0..2] are reused for partials B iterations on
        }
    } else {
        gamma = cur[0];
        delta = cur[1];
        rr = cur[2];
    }
    bool stopping = false;
    // peer all-reduce: ||r_0||^2 is known only here, at the first step (k = 0)
    const bool first = rg.win && (ctl ? ctl[2] == 0 : prev[0] == 0.0);
    const double rr0v = tol < 0.0 ? 0.0 : (first ? rr : rr0[0]);
    if (first && rr0 && blockIdx.x == 0 && threadIdx.x == 0) rr0[0] = rr;
    if (ctl) {
        const double nk = sqrt(rr);
        const bool bad = !isfinite(nk);
        if (bad || (tol >= 0.0 && nk <= tol * sqrt(rr0v))) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                ctl[1] = ctl[2];
                ctl[3] = bad ? 1 : 0;
                ctl[0] = 1;
            }
            // every block takes the same decision from the same scalars
            if (!rg.win) return;
            stopping = true;
        }
    }
    const double g_prev = prev[0], a_prev = prev[3];
    const double beta = g_prev != 0.0 ? gamma / g_prev : 0.0;
    const double denom = (beta != 0.0 && a_prev != 0.0) ? delta - beta * gamma / a_prev : delta;
    const double alpha = denom != 0.0 ? gamma / denom : 0.0;
    double part[2] = {0.0, 0.0};
    bool bad = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < (stopping ? 0 : n);
         base += stride * VEC_ILP) {
        double uv[VEC_ILP], wv[VEC_ILP], pv[VEC_ILP], sv[VEC_ILP], xv[VEC_ILP], rv[VEC_ILP],
            dv[VEC_ILP];
        uint8_t ow[VEC_ILP];
#pragma unroll
        for (int q = 0; q < VEC_ILP; ++q) {
            const int64_t m = base + q * stride;
            const bool ok = m < n;
            uv[q] = ok ? u[m] : 0.0;
            wv[q] = ok ? w[m] : 0.0;
            pv[q] = ok ? p[m] : 0.0;
            sv[q] = ok ? s[m] : 0.0;
            xv[q] = ok ? x[m] : 0.0;
            rv[q] = ok ? r[m] : 0.0;
            dv[q] = ok ? dinv[m] : 0.0;
            ow[q] = ok ? owned[m] : 0;
        }
#pragma unroll
        for (int q = 0; q < VEC_ILP; ++q) {
            const int64_t m = base + q * stride;
            if (m < n) {
                const double pn = uv[q] + beta * pv[q];
                const double sn = wv[q] + beta * sv[q];
                const double xn = xv[q] + alpha * pn;
                const double rn = rv[q] - alpha * sn;
                const double un = dv[q] * rn;
                p[m] = pn;
                s[m] = sn;
                x[m] = xn;
                r[m] = rn;
                u[m] = un;
                bad |= !isfinite(xn);
                if (ow[q]) {
                    part[0] += rn * un;
                    part[1] += rn * rn;
                }
            }
        }
    }
    if (bad) atomicOr(nonfinite, 1);
    double tot[2];
    if (grid_sum_last<2>(part, partials, counter, tot) && threadIdx.x == 0) {
        if (rg.win) reinterpret_cast<WinHdr *>(rg.win)->red_epoch = ep + 1;
        if (hr.hdr) hr.hdr->done_a = 0;  // every block is past the barrier
        if (!stopping) {
            next[0] = tot[0];
            next[2] = tot[1];
            cur[3] = alpha;
            if (ctl) ctl[2] += 1;
        }
    }
}

// red[0] = sum_owned x*y (owned nullable: all)
__global__ void __launch_bounds__(256)
    k_vec_dot_owned(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                    const uint8_t *__restrict__ owned, double *partials, unsigned int *counter,
                    double *red) {
    double part[1] = {0.0};
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x)
        if (!owned || owned[m]) part[0] += x[m] * y[m];
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

// dinv = free ? (diag ? (diag != 0 ? 1/diag : 0) : 1) : 0
__global__ void k_vec_dinv(int64_t n, const double *__restrict__ diag,
                           const uint8_t *__restrict__ free_m, double *__restrict__ dinv) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x)
        dinv[m] = free_m[m] ? (diag ? (diag[m] != 0.0 ? 1.0 / diag[m] : 0.0) : 1.0) : 0.0;
}

struct Scratch {
    double *partials;
    unsigned int *counter;
};

static Scratch scratch(void *ws) {
    // ws: caller-provided device workspace of ebs_vec_workspace_bytes() bytes
    Scratch s;
    s.counter = reinterpret_cast<unsigned int *>(ws);
    s.partials = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + 256);
    return s;
}

}  // namespace ebs

namespace ebs {
// the same step with cur[0..2] all-reduced on the device from the peer window (ebs_peer_*)
int peer_cg1_update(const ebs::RedGet &rg, const ebs::PeerRecv &hr, const uint8_t *free_m,
                    int64_t n, double *cur, const double *prev,
                    const double *rr0, double tol, int32_t *ctl, const uint8_t *owned,
                    const double *dinv, double *x, double *r, double *u, const double *w,
                    double *p, double *s, double *next, int32_t *nonfinite, void *ws,
                    void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && cur && prev && owned && dinv && x && r && u && w && p && s && next &&
                    nonfinite && ws && (rr0 || tol < 0.0) && rg.win,
                "null argument");
    Scratch sc = scratch(ws);
    const int grid = persistent_grid((const void *)k_vec_cg1_update, 256, (n + 255) / 256, 0);
    k_vec_cg1_update<<<grid, 256, 0, S(stream)>>>(
        n, cur, prev, const_cast<double *>(rr0), tol, ctl, owned, dinv, x, r, u,
        const_cast<double *>(w), p, s, sc.partials, sc.counter, next, nonfinite, rg, hr,
        free_m);
    LAUNCHED();
    EBS_CATCH
}

}  // namespace ebs

using namespace ebs;

extern "C" {

size_t ebs_vec_workspace_bytes(void) { return 256 + sizeof(double) * 2 * 8192; }

int ebs_index_fill(int64_t n, const int64_t *idx, double value, double *v, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "bad n");
    if (n == 0) return EBS_OK;
    k_index_fill<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, idx, value, v);
    LAUNCHED();
    EBS_CATCH
}

int ebs_index_copy(int64_t n, const int64_t *idx, const double *src, double *dst, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "bad n");
    if (n == 0) return EBS_OK;
    k_index_copy<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, idx, src, dst);
    LAUNCHED();
    EBS_CATCH
}

int ebs_index_move(int64_t n, const int64_t *src_idx, const double *src, const int64_t *dst_idx,
                   double *dst, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "bad n");
    if (n == 0) return EBS_OK;
    k_index_move<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, src_idx, src, dst_idx, dst);
    LAUNCHED();
    EBS_CATCH
}

int ebs_index_add(int64_t n, const int64_t *src_idx, const double *src, const int64_t *dst_idx,
                  double *dst, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "bad n");
    if (n == 0) return EBS_OK;
    k_index_add<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, src_idx, src, dst_idx, dst);
    LAUNCHED();
    EBS_CATCH
}

int ebs_vec_jacobi(int64_t n, double omega, const double *b, const double *s, const double *dinv,
                   const uint8_t *free_m, const uint8_t *owned, const double *x, double *x_out,
                   double *r_out, double *red, int32_t *nonfinite, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && b && s && free_m && owned && red && nonfinite && ws, "null argument");
    EBS_REQUIRE(!x_out || x, "x_out needs x");
    Scratch sc = scratch(ws);
    k_vec_jacobi<<<grid_for(n, 256, RED_MAX_BLOCKS), 256, 0, S(stream)>>>(
        n, omega, b, s, dinv, free_m, owned, x, x_out, r_out, sc.partials, sc.counter, red,
        nonfinite);
    LAUNCHED();
    EBS_CATCH
}

int ebs_vec_pcg_q(int64_t n, const uint8_t *free_m, const uint8_t *owned, const double *p,
                  double *q, double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && free_m && owned && p && q && red && ws, "null argument");
    Scratch sc = scratch(ws);
    k_vec_pcg_q<<<grid_for(n, 256, RED_MAX_BLOCKS), 256, 0, S(stream)>>>(
        n, free_m, owned, p, q, sc.partials, sc.counter, red);
    LAUNCHED();
    EBS_CATCH
}

int ebs_vec_pcg_update(int64_t n, const double *rz, const double *pq, const uint8_t *owned,
                       const double *dinv, double *x, double *r, const double *p, const double *q,
                       double *red, int32_t *nonfinite, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && rz && pq && owned && dinv && x && r && p && q && red && nonfinite && ws,
                "null argument");
    Scratch sc = scratch(ws);
    // one wave of resident CTAs (occupancy-sized, fixed per device: deterministic order);
    // the capped 1184-CTA grid ran in 4 waves at these kernels' register counts
    const int grid = persistent_grid((const void *)k_vec_pcg_update, 256, (n + 255) / 256, 0);
    k_vec_pcg_update<<<grid, 256, 0, S(stream)>>>(
        n, rz, pq, owned, dinv, x, r, p, q, sc.partials, sc.counter, red, nonfinite);
    LAUNCHED();
    EBS_CATCH
}

int ebs_vec_pcg_direction(int64_t n, const double *rz_old, const double *rz_new,
                          const double *dinv, const double *r, double *p, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && rz_old && rz_new && dinv && r && p, "null argument");
    if (n == 0) return EBS_OK;
    k_vec_pcg_direction<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, rz_old, rz_new, dinv, r, p);
    LAUNCHED();
    EBS_CATCH
}

int ebs_vec_cg1_update(int64_t n, double *cur, const double *prev, const double *rr0, double tol,
                       int32_t *ctl, const uint8_t *owned, const double *dinv, double *x,
                       double *r, double *u, const double *w, double *p, double *s,
                       double *next, int32_t *nonfinite, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && cur && prev && owned && dinv && x && r && u && w && p && s && next &&
                    nonfinite && ws && (rr0 || tol < 0.0),
                "null argument");
    Scratch sc = scratch(ws);
    const int grid = persistent_grid((const void *)k_vec_cg1_update, 256, (n + 255) / 256, 0);
    k_vec_cg1_update<<<grid, 256, 0, S(stream)>>>(
        n, cur, prev, const_cast<double *>(rr0), tol, ctl, owned, dinv, x, r, u,
        const_cast<double *>(w), p, s, sc.partials, sc.counter, next, nonfinite,
        RedGet{nullptr, 0, 0}, PeerRecv{}, nullptr);
    LAUNCHED();
    EBS_CATCH
}

int ebs_dist_set_stop(ebs_plan_t plan, const int32_t *stop) {
    EBS_TRY
    EBS_REQUIRE(plan, "null argument");
    reinterpret_cast<Plan *>(plan)->dist_stop = stop;
    EBS_CATCH
}

int ebs_vec_dot_owned(int64_t n, const double *x, const double *y, const uint8_t *owned,
                      double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && x && y && red && ws, "null argument");
    Scratch sc = scratch(ws);
    k_vec_dot_owned<<<grid_for(n, 256, RED_MAX_BLOCKS), 256, 0, S(stream)>>>(
        n, x, y, owned, sc.partials, sc.counter, red);
    LAUNCHED();
    EBS_CATCH
}

int ebs_vec_dinv(int64_t n, const double *diag, const uint8_t *free_m, double *dinv,
                 void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && free_m && dinv, "null argument");
    if (n == 0) return EBS_OK;
    k_vec_dinv<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, diag, free_m, dinv);
    LAUNCHED();
    EBS_CATCH
}

int ebs_plan_free_mask(ebs_plan_t plan, uint8_t *free_int, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && free_int, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (p->n_n)
        CU(cudaMemcpyAsync(free_int, p->free_int, p->n_n, cudaMemcpyDeviceToDevice, S(stream)));
    EBS_CATCH
}

int ebs_plan_internal_rhs(ebs_plan_t plan, double *b_int, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && b_int, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_be, "no b_e loaded");
    if (p->n_n)
        CU(cudaMemcpyAsync(b_int, p->b_int, sizeof(double) * p->n_n, cudaMemcpyDeviceToDevice,
                           S(stream)));
    EBS_CATCH
}

}  // extern "C"

// ------------------------------------------------------------------------------------
// Fused slab-rank steps.  The SELL sweep covers a chunk list; nodes flagged `iface` (shared
// with another slab) only store their partial sum for the halo exchange, all other nodes
// (owned, complete) are finished in the epilogue exactly as the 1-GPU fused kernels do.
// Sweeping the interface chunks first lets the host start the exchange while the
// interior chunks are swept.
#include "sell.cuh"

namespace ebs {

struct DistJacobiEpi {
    double omega;
    const double *__restrict__ b;
    const double *__restrict__ dinv;
    const uint8_t *__restrict__ free_m;
    const uint8_t *__restrict__ iface;
    double *__restrict__ x_out;
    double *__restrict__ s_part;
    double part[1];
    __device__ __forceinline__ void operator()(int64_t m, double s, double xo) {
        if (iface[m]) {
            s_part[m] = s;
            return;
        }
        double r = free_m[m] ? b[m] - s : 0.0;
        part[0] += r * r;
        if (x_out) x_out[m] = dinv ? xo + omega * (dinv[m] * r) : xo + omega * r;
    }
};

template <int NB, int IDS>
__global__ void EBS_SELL_BOUNDS(NB)
    k_dist_jacobi_sweep(SellView v, const double *__restrict__ x, DistJacobiEpi epi,
                        double *partials, unsigned int *counter, double *red) {
    sell_sweep<NB, IDS, false, NB == 3>(v, x, epi);
    double tot[1];
    if (grid_sum_last<1>(epi.part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

struct DistMatvecEpi {
    const uint8_t *__restrict__ free_m;
    const uint8_t *__restrict__ iface;
    double *__restrict__ q;
    double part[1];
    __device__ __forceinline__ void operator()(int64_t m, double s, double po) {
        if (iface[m]) {
            q[m] = s;  // partial; completed after the halo
            return;
        }
        double qm = free_m[m] ? s : 0.0;
        q[m] = qm;
        part[0] += po * qm;
    }
};

template <int NB, int IDS>
__global__ void EBS_SELL_BOUNDS(NB)
    k_dist_matvec_sweep(SellView v, const double *__restrict__ p, DistMatvecEpi epi,
                        double *partials, unsigned int *counter, double *red,
                        const int32_t *stop) {
    if (stop && *stop) return;  // single-reduction PCG already stopped (ebs_dist_set_stop)
    sell_sweep<NB, IDS, false>(v, p, epi);
    double tot[1];
    if (grid_sum_last<1>(epi.part, partials, counter, tot) && threadIdx.x == 0) red[0] = tot[0];
}

// interface nodes after the halo: Jacobi completion (s combined) / PCG q completion
__global__ void __launch_bounds__(256)
    k_dist_jacobi_iface(int64_t n, const int64_t *__restrict__ idx, double omega,
                        const double *__restrict__ b, const double *__restrict__ s,
                        const double *__restrict__ dinv, const uint8_t *__restrict__ free_m,
                        const uint8_t *__restrict__ owned, const double *__restrict__ x,
                        double *__restrict__ x_out, double *partials, unsigned int *counter,
                        const double *prior, double *red) {
    double part[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = idx[i];
        double r = free_m[m] ? b[m] - s[m] : 0.0;
        if (owned[m]) part[0] += r * r;
        if (x_out) x_out[m] = dinv ? x[m] + omega * (dinv[m] * r) : x[m] + omega * r;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0)
        red[0] = prior ? (prior[0] + prior[1]) + tot[0] : tot[0];
}

__global__ void __launch_bounds__(256)
    k_dist_q_iface(int64_t n, const int64_t *__restrict__ idx, const uint8_t *__restrict__ free_m,
                   const uint8_t *__restrict__ owned, const double *__restrict__ p,
                   double *__restrict__ q, double *partials, unsigned int *counter,
                   const double *prior, double *red) {
    double part[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = idx[i];
        double qm = free_m[m] ? q[m] : 0.0;
        q[m] = qm;
        if (owned[m]) part[0] += p[m] * qm;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0)
        red[0] = prior ? (prior[0] + prior[1]) + tot[0] : tot[0];
}

// v[m] = sum of the contributions to shared node m, in ascending rank order (the own
// partial among them): one thread per interface node, sources by value (<= COMBINE_MAX;
// geometric slabs have 2 neighbours, thin ones a few more), pos[i * n_src + k] = index of node i in source k or -1.  Replaces a
// fill, a gather and one scatter-add per source with one pass (same order of additions).
constexpr int COMBINE_MAX = 8;
struct CombineSrc {
    const double *p[COMBINE_MAX];
    int n;
};

__global__ void __launch_bounds__(256)
    k_dist_combine(int64_t n_if, const int64_t *__restrict__ all_if, CombineSrc src,
                   const int32_t *__restrict__ pos, double *v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = all_if[i];
        double acc = 0.0;
        for (int k = 0; k < src.n; ++k) {
            const int32_t q = pos[i * src.n + k];
            if (q >= 0) acc += src.p[k][q];
        }
        v[m] = acc;
    }
}

// The combine and the interface completion in one pass (one launch less per iteration on
// the latency-bound halo tail): thread i sums the contributions to shared node all_if[i] in
// ascending rank order (as k_dist_combine) and completes that node at once (as
// k_dist_jacobi_iface / k_dist_q_iface) -- each thread reads and writes only its own node.
__global__ void __launch_bounds__(256)
    k_dist_combine_jacobi(int64_t n_if, const int64_t *__restrict__ all_if, CombineSrc src,
                          const int32_t *__restrict__ pos, double *s, double omega,
                          const double *__restrict__ b, const double *__restrict__ dinv,
                          const uint8_t *__restrict__ free_m, const uint8_t *__restrict__ owned,
                          const double *__restrict__ x, double *__restrict__ x_out,
                          double *partials, unsigned int *counter, const double *prior,
                          double *red) {
    double part[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = all_if[i];
        double acc = 0.0;
        for (int k = 0; k < src.n; ++k) {
            const int32_t q = pos[i * src.n + k];
            if (q >= 0) acc += src.p[k][q];
        }
        s[m] = acc;
        const double r = free_m[m] ? b[m] - acc : 0.0;
        if (owned[m]) part[0] += r * r;
        if (x_out) x_out[m] = dinv ? x[m] + omega * (dinv[m] * r) : x[m] + omega * r;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0)
        red[0] = prior ? (prior[0] + prior[1]) + tot[0] : tot[0];
}

__global__ void __launch_bounds__(256)
    k_dist_combine_q(int64_t n_if, const int64_t *__restrict__ all_if, CombineSrc src,
                     const int32_t *__restrict__ pos, double *q, const uint8_t *__restrict__ free_m,
                     const uint8_t *__restrict__ owned, const double *__restrict__ p,
                     double *partials, unsigned int *counter, const double *prior, double *red) {
    double part[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_if;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = all_if[i];
        double acc = 0.0;
        for (int k = 0; k < src.n; ++k) {
            const int32_t c = pos[i * src.n + k];
            if (c >= 0) acc += src.p[k][c];
        }
        const double qm = free_m[m] ? acc : 0.0;
        q[m] = qm;
        if (owned[m]) part[0] += p[m] * qm;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0)
        red[0] = prior ? (prior[0] + prior[1]) + tot[0] : tot[0];
}

}  // namespace ebs

extern "C" {

int ebs_dist_jacobi_sweep(ebs_plan_t plan, const int32_t *chunks, int64_t n_list, double omega,
                          const double *x, double *x_out, const double *b, const double *dinv,
                          const uint8_t *iface, double *s_part, double *red, void *ws,
                          void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x && b && iface && s_part && red && ws, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(n_list >= 0 && (chunks || n_list == 0), "bad chunk list");
    Scratch sc = scratch(ws);
    if (n_list == 0) {
        CU(cudaMemsetAsync(red, 0, sizeof(double), S(stream)));
        return EBS_OK;
    }
    DistJacobiEpi epi{omega, b, dinv, p->free_int, iface, x_out, s_part, {0.0}};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_DJ(NB_, IDS_)                                                                   \
    {                                                                                       \
        auto kern = k_dist_jacobi_sweep<NB_, IDS_>;                                         \
        SellLaunch SL = sell_launch((const void *)kern, NB_, p->rowb, n_list);              \
        kern<<<SL.grid, SL.block, SL.smem, S(stream)>>>(v, x, epi, sc.partials, sc.counter, \
                                                        red);                               \
    }
    EBS_SELL_DISPATCH(p, EBS_DJ);
#undef EBS_DJ
    LAUNCHED();
    EBS_CATCH
}

int ebs_dist_matvec_sweep(ebs_plan_t plan, const int32_t *chunks, int64_t n_list, const double *pv,
                          double *q, const uint8_t *iface, double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && pv && q && iface && red && ws, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(n_list >= 0 && (chunks || n_list == 0), "bad chunk list");
    Scratch sc = scratch(ws);
    if (n_list == 0) {
        CU(cudaMemsetAsync(red, 0, sizeof(double), S(stream)));
        return EBS_OK;
    }
    DistMatvecEpi epi{p->free_int, iface, q, {0.0}};
    SellView v = sell_view(p, chunks, n_list);
#define EBS_DM(NB_, IDS_)                                                                   \
    {                                                                                       \
        auto kern = k_dist_matvec_sweep<NB_, IDS_>;                                         \
        SellLaunch SL = sell_launch((const void *)kern, NB_, p->rowb, n_list);              \
        kern<<<SL.grid, SL.block, SL.smem, S(stream)>>>(v, pv, epi, sc.partials, sc.counter, \
                                                        red, p->dist_stop);                 \
    }
    EBS_SELL_DISPATCH(p, EBS_DM);
#undef EBS_DM
    LAUNCHED();
    EBS_CATCH
}

int ebs_dist_jacobi_iface(int64_t n, const int64_t *idx, double omega, const double *b,
                          const double *s, const double *dinv, const uint8_t *free_m,
                          const uint8_t *owned, const double *x, double *x_out,
                          const double *prior, double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && b && s && free_m && owned && x && red && ws, "null argument");
    Scratch sc = scratch(ws);
    k_dist_jacobi_iface<<<grid_for(n, 256, RED_MAX_BLOCKS), 256, 0, S(stream)>>>(
        n, idx, omega, b, s, dinv, free_m, owned, x, x_out, sc.partials, sc.counter, prior, red);
    LAUNCHED();
    EBS_CATCH
}

int ebs_dist_combine(int64_t n_if, const int64_t *all_if, int n_src, const double *const *srcs,
                     const int32_t *pos, double *v, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n_if >= 0 && n_src >= 1 && n_src <= COMBINE_MAX && srcs &&
                    (n_if == 0 || (all_if && pos && v)),
                "bad arguments (1 <= n_src <= %d)", COMBINE_MAX);
    if (n_if == 0) return EBS_OK;
    CombineSrc cs{};
    cs.n = n_src;
    for (int k = 0; k < n_src; ++k) {
        EBS_REQUIRE(srcs[k], "null source %d", k);
        cs.p[k] = srcs[k];
    }
    k_dist_combine<<<grid_for(n_if, 256), 256, 0, S(stream)>>>(n_if, all_if, cs, pos, v);
    LAUNCHED();
    EBS_CATCH
}

int ebs_dist_q_iface(int64_t n, const int64_t *idx, const uint8_t *free_m, const uint8_t *owned,
                     const double *pv, double *q, const double *prior, double *red, void *ws,
                     void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && free_m && owned && pv && q && red && ws, "null argument");
    Scratch sc = scratch(ws);
    k_dist_q_iface<<<grid_for(n, 256, RED_MAX_BLOCKS), 256, 0, S(stream)>>>(
        n, idx, free_m, owned, pv, q, sc.partials, sc.counter, prior, red);
    LAUNCHED();
    EBS_CATCH
}


static CombineSrc combine_sources(int n_src, const double *const *srcs) {
    EBS_REQUIRE(n_src >= 1 && n_src <= COMBINE_MAX && srcs, "1 <= n_src <= %d sources",
                COMBINE_MAX);
    CombineSrc cs{};
    cs.n = n_src;
    for (int k = 0; k < n_src; ++k) {
        EBS_REQUIRE(srcs[k], "null source %d", k);
        cs.p[k] = srcs[k];
    }
    return cs;
}

int ebs_dist_combine_jacobi(int64_t n_if, const int64_t *all_if, int n_src,
                            const double *const *srcs, const int32_t *pos, double *s, double omega,
                            const double *b, const double *dinv, const uint8_t *free_m,
                            const uint8_t *owned, const double *x, double *x_out,
                            const double *prior, double *red, void *ws, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n_if >= 0 && s && b && free_m && owned && x && red && ws &&
                    (n_if == 0 || (all_if && pos)),
                "null argument");
    const CombineSrc cs = combine_sources(n_src, srcs);
    Scratch sc = scratch(ws);
    const int grid = persistent_grid((const void *)k_dist_combine_jacobi, 256, (n_if + 255) / 256, 0);
    k_dist_combine_jacobi<<<grid, 256, 0, S(stream)>>>(n_if, all_if, cs, pos, s, omega, b, dinv,
                                                       free_m, owned, x, x_out, sc.partials,
                                                       sc.counter, prior, red);
    LAUNCHED();
    EBS_CATCH
}

int ebs_dist_combine_q(int64_t n_if, const int64_t *all_if, int n_src, const double *const *srcs,
                       const int32_t *pos, double *q, const uint8_t *free_m, const uint8_t *owned,
                       const double *pv, const double *prior, double *red, void *ws,
                       void *stream) {
    EBS_TRY
    EBS_REQUIRE(n_if >= 0 && q && free_m && owned && pv && red && ws &&
                    (n_if == 0 || (all_if && pos)),
                "null argument");
    const CombineSrc cs = combine_sources(n_src, srcs);
    Scratch sc = scratch(ws);
    const int grid = persistent_grid((const void *)k_dist_combine_q, 256, (n_if + 255) / 256, 0);
    k_dist_combine_q<<<grid, 256, 0, S(stream)>>>(n_if, all_if, cs, pos, q, free_m, owned, pv,
                                                  sc.partials, sc.counter, prior, red);
    LAUNCHED();
    EBS_CATCH
}

}  // extern "C"

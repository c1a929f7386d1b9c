// solve.cu -- the solvers.py:117-160 `_iterate` loop run on the device.
//
// Richardson / damped Jacobi (one fused launch per iteration):
//   L(k): r_k = mask(b - A x_k) [SELL]; ||r_k||^2 (+ ||x_k - ref||^2) reduced in-kernel;
//         x_{k+1} = x_k + omega*r_k   (Richardson, solvers.py:179-180)
//         x_{k+1} = x_k + omega*(dinv*r_k)   (Jacobi)
//         into the other ping-pong buffer.  The last CTA applies the loop rules:
//         record norms[k]; k>0 and non-finite -> diverged (solvers.py:150-152);
//         ||r_k|| <= tol*||r_0|| -> stop with x_k (solvers.py:135);
//         x_{k+1} non-finite -> norms[k+1] = inf, diverged (solvers.py:138-143).
//   R   : the residual of the last iterate (history entry `iters`).
// CG / Jacobi-PCG (oracle/ebs_oracle.py pcg): init I, then per iteration
//   M(k): q = mask(A p) [SELL] + p.q  -> alpha
//   U(k): x += alpha p, r -= alpha q, ||r||^2, r.(dinv r) -> norms[k+1], beta
//   P(k): p = dinv*r + beta*p
// Kernels read the iteration index and the stop flag from the device control block, so
// the host only enqueues launches; it synchronises once per batch of iterations to stop
// enqueuing after convergence (and every iteration when a callback is attached).
// Reductions are fixed-order (deterministic run to run).
#include <cooperative_groups.h>
#include <cstdlib>
#include <vector>

#include "sell.cuh"

namespace ebs {


struct LoopArgs {
    Ctl *ctl;
    double *norms;   // device history
    double *errors;  // device history (nullable)
    double *partials;
    int has_tol;
    double tol;
    double omega;
};

__device__ __forceinline__ void flag_nonfinite(Ctl *ctl, bool bad) {
    if (bad) {
        atomicOr(&ctl->nonfinite, 1);
        __threadfence();
    }
}

// ---------------------------------------------------------- Richardson/Jacobi --
// stationary steps on the _iterate loop, KIND (template) x method:
//   JK_PLAIN  x + omega*r       Richardson (omega), Chebyshev-2 (omega = a_k)
//   JK_JACOBI x + omega*(dinv*r)
//   JK_CHEB3  p = k ? r + b_k*p : r;  x + a_k*p
// The loop-invariant pointers come from a __grid_constant__ argument block (read from
// the constant bank where used, never held in registers): with the per-method template
// the 2D kernels fit the 32-register cap of 64 warps/SM without spilling.
constexpr int JK_PLAIN = 0, JK_JACOBI = 1, JK_CHEB3 = 2;

struct JacArgs {
    const double *b_int;
    const uint8_t *free_int;
    const double *dinv;
    const double *ref;
    double *r_out;
    double *xa, *xb;
    double *pbuf;
    const double *ca, *cb;
    int final_step;
};

template <int KIND, bool EXACT>
struct JacobiEpi {
    const JacArgs &A;
    const LoopArgs &L;
    double part[1];
    __device__ __forceinline__ void operator()(int64_t m, double s, double xo) {
        double r = EXACT ? s : A.b_int[m] - s;
        if (!A.free_int[m]) r = 0.0;
        part[0] += r * r;
        if (A.r_out) A.r_out[m] = r;
        if (!A.final_step) {
            // the step's scalars are re-read here (L1 / constant-bank hits) instead of
            // being carried in registers across the sweep: no spills at 32 registers
            const int k = __ldg(&L.ctl->k);
            double *xn_buf = (k & 1) ? A.xa : A.xb;
            double xn;
            if constexpr (KIND == JK_JACOBI) {
                xn = xo + L.omega * (A.dinv[m] * r);
            } else if constexpr (KIND == JK_CHEB3) {
                const double om = __ldg(A.ca + k);
                double pm = k == 0 ? r : r + __ldg(A.cb + k) * A.pbuf[m];
                A.pbuf[m] = pm;
                xn = xo + om * pm;
            } else {
                const double om = A.ca ? __ldg(A.ca + k) : L.omega;
                xn = xo + om * r;
            }
            xn_buf[m] = xn;
            if (!isfinite(xn)) flag_nonfinite(L.ctl, true);  // rare: no per-thread flag
        }
    }
};

// ||x_k - ref||^2 of the iterate step k reads (the stationary loop with a reference
// solution, solvers.py:146-148): its own fixed-order reduction, launched before the step,
// so the step kernel carries one accumulator (no spills at the 2D register cap).
__global__ void __launch_bounds__(256)
    k_err_norm(int64_t n, LoopArgs L, const double *__restrict__ xa,
               const double *__restrict__ xb, const double *__restrict__ ref) {
    Ctl *ctl = L.ctl;
    if (ctl->done) return;
    const int k = ctl->k;
    const double *x = (k & 1) ? xb : xa;
    double part[1] = {0.0};
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        const double d = x[m] - ref[m];
        part[0] += d * d;
    }
    double tot[1];
    if (grid_sum_last<1>(part, L.partials, &ctl->counter, tot) && threadIdx.x == 0)
        L.errors[k] = sqrt(tot[0]);
}

#ifndef EBS_JAC_MINB2
#define EBS_JAC_MINB2 EBS_MINB2
#endif
#ifndef EBS_JAC_PIPE
#define EBS_JAC_PIPE 1
#endif
template <int NB, int IDS, bool EXACT, int KIND>
__global__ void __launch_bounds__(256, (NB) == 3 ? EBS_JAC_MINB2 : EBS_MINB3)
    k_jacobi_step(SellView v, const __grid_constant__ LoopArgs L,
                  const __grid_constant__ JacArgs A) {
    Ctl *ctl = L.ctl;
    if (ctl->done) return;
    const int k = ctl->k;
    JacobiEpi<KIND, EXACT> epi{A, L, {0.0}};
    sell_sweep<NB, IDS, EXACT, NB == 3 && EBS_JAC_PIPE>(v, (k & 1) ? A.xb : A.xa, epi);
    double tot[1];
    if (!grid_sum_last<1>(epi.part, L.partials, &ctl->counter, tot) || threadIdx.x != 0) return;
    // ---- loop rules (single thread) ----
    __threadfence();  // the rare non-finite flags of this grid (flag_nonfinite) are visible
    const double nr = sqrt(tot[0]);
    L.norms[k] = nr;
    if (k == 0) ctl->norm0 = nr;
    ctl->n_norms = k + 1;
    ctl->cb_ok = 1;
    ctl->final_buf = k & 1;
    if (k > 0 && !isfinite(nr)) {
        ctl->diverged = 1;
        ctl->done = 1;
        return;
    }
    if (A.final_step) {
        ctl->done = 1;
        return;
    }
    if (L.has_tol && nr <= L.tol * ctl->norm0) {
        ctl->done = 1;
        return;
    }
    if (ctl->nonfinite) {
        L.norms[k + 1] = INFINITY;
        if (L.errors) L.errors[k + 1] = INFINITY;
        ctl->n_norms = k + 2;
        ctl->diverged = 1;
        ctl->done = 1;
        ctl->final_buf = (k + 1) & 1;
        ctl->k = k + 1;
        return;
    }
    ctl->k = k + 1;
    ctl->final_buf = (k + 1) & 1;
}

// ------------------------------------------------------------------ CG / PCG --
struct PcgInitEpi {
    const double *__restrict__ b_int;
    const uint8_t *__restrict__ free_int;
    const double *__restrict__ dinv;
    const double *__restrict__ ref;
    double *__restrict__ r_int;
    double *__restrict__ p_int;
    double part[3];
    __device__ __forceinline__ void operator()(int64_t m, double s, double xo) {
        double r = free_int[m] ? b_int[m] - s : 0.0;
        double z = dinv[m] * r;
        r_int[m] = r;
        p_int[m] = z;
        part[0] += r * r;
        part[1] += r * z;
        if (ref) {
            double d = xo - ref[m];
            part[2] += d * d;
        }
    }
};

template <int NB, int IDS>
__global__ void EBS_SELL_BOUNDS(NB)
    k_pcg_init(SellView v, LoopArgs L, const double *__restrict__ x, PcgInitEpi epi) {
    Ctl *ctl = L.ctl;
    sell_sweep<NB, IDS, false>(v, x, epi);
    double tot[3];
    if (!grid_sum_last<3>(epi.part, L.partials, &ctl->counter, tot) || threadIdx.x != 0) return;
    const double nr = sqrt(tot[0]);
    L.norms[0] = nr;
    if (L.errors) L.errors[0] = sqrt(tot[2]);
    ctl->norm0 = nr;
    ctl->rz = tot[1];
    ctl->n_norms = 1;
    ctl->k = 0;
    ctl->cb_ok = 1;
    if (L.has_tol && nr <= L.tol * nr) ctl->done = 1;
}

struct PcgMatvecEpi {
    const uint8_t *__restrict__ free_int;
    double *__restrict__ q_int;
    double part[1];
    __device__ __forceinline__ void operator()(int64_t m, double s, double po) {
        double q = free_int[m] ? s : 0.0;  // spectrum.py:60 out[nd] = 0
        q_int[m] = q;
        part[0] += po * q;
    }
};

template <int NB, int IDS>
__global__ void EBS_SELL_BOUNDS(NB)
    k_pcg_matvec(SellView v, LoopArgs L, const double *__restrict__ p_int, PcgMatvecEpi epi) {
    Ctl *ctl = L.ctl;
    if (ctl->done) return;
    sell_sweep<NB, IDS, false>(v, p_int, epi);
    double tot[1];
    if (!grid_sum_last<1>(epi.part, L.partials, &ctl->counter, tot) || threadIdx.x != 0) return;
    ctl->pq = tot[0];
    ctl->alpha = tot[0] != 0.0 ? ctl->rz / tot[0] : 0.0;
}

#ifndef EBS_UPD_MINB
#define EBS_UPD_MINB 3
#endif
#ifndef EBS_UPD_PERSIST
#define EBS_UPD_PERSIST 1  // occupancy-sized grid, one wave (C3: 2775 -> 2824 it/s vs 1184 CTAs)
#endif
__global__ void __launch_bounds__(256, EBS_UPD_MINB)
    k_pcg_update(int64_t n, LoopArgs L, double *__restrict__ x, double *__restrict__ r,
                 const double *__restrict__ p, const double *__restrict__ q,
                 const double *__restrict__ dinv, const double *__restrict__ ref) {
    Ctl *ctl = L.ctl;
    if (ctl->done) return;
    const double alpha = ctl->alpha;
    double part[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    constexpr int ILP = 4;  // independent node updates in flight per thread
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n;
         base += stride * ILP) {
        double xv[ILP], rv[ILP], pv[ILP], qv[ILP], dv[ILP], fv[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t m = base + u * stride;
            const bool ok = m < n;
            xv[u] = ok ? x[m] : 0.0;
            rv[u] = ok ? r[m] : 0.0;
            pv[u] = ok ? p[m] : 0.0;
            qv[u] = ok ? q[m] : 0.0;
            dv[u] = ok ? dinv[m] : 0.0;
            fv[u] = (ok && ref) ? ref[m] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t m = base + u * stride;
            if (m < n) {
                double xn = xv[u] + alpha * pv[u];
                double rn = rv[u] - alpha * qv[u];
                x[m] = xn;
                r[m] = rn;
                bad |= !isfinite(xn);
                part[0] += rn * rn;
                part[1] += rn * (dv[u] * rn);
                if (ref) {
                    double d = xn - fv[u];
                    part[2] += d * d;
                }
            }
        }
    }
    flag_nonfinite(ctl, bad);
    double tot[3];
    if (!grid_sum_last<3>(part, L.partials, &ctl->counter, tot) || threadIdx.x != 0) return;
    const int k = ctl->k;
    ctl->k = k + 1;
    ctl->n_norms = k + 2;
    if (ctl->nonfinite) {
        L.norms[k + 1] = INFINITY;
        if (L.errors) L.errors[k + 1] = INFINITY;
        ctl->diverged = 1;
        ctl->done = 1;
        ctl->cb_ok = 0;
        return;
    }
    const double nr = sqrt(tot[0]);
    L.norms[k + 1] = nr;
    if (L.errors) L.errors[k + 1] = sqrt(tot[2]);
    ctl->cb_ok = 1;
    if (!isfinite(nr)) {
        ctl->diverged = 1;
        ctl->done = 1;
        return;
    }
    if (L.has_tol && nr <= L.tol * ctl->norm0) {
        ctl->done = 1;
        return;
    }
    const double rz_new = tot[1];
    ctl->beta = ctl->rz != 0.0 ? rz_new / ctl->rz : 0.0;
    ctl->rz = rz_new;
}

__global__ void __launch_bounds__(256)
    k_pcg_direction(int64_t n, Ctl *ctl, double *__restrict__ p, const double *__restrict__ r,
                    const double *__restrict__ dinv) {
    if (ctl->done) return;
    const double beta = ctl->beta;
    constexpr int ILP = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n;
         base += stride * ILP) {
        double rv[ILP], pv[ILP], dv[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t m = base + u * stride;
            const bool ok = m < n;
            rv[u] = ok ? r[m] : 0.0;
            pv[u] = ok ? p[m] : 0.0;
            dv[u] = ok ? dinv[m] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t m = base + u * stride;
            if (m < n) p[m] = dv[u] * rv[u] + beta * pv[u];
        }
    }
}

// dinv = 1/diag on free nodes (Jacobi, PCG), 1 on free nodes (CG), 0 on constrained
// nodes and on nodes no element touches (diag == 0: no equation, the iterate stays put)
__global__ void k_dinv(int64_t n, const double *__restrict__ diag,
                       const uint8_t *__restrict__ free_int, double *__restrict__ dinv) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x)
        dinv[m] = free_int[m] ? (diag ? (diag[m] != 0.0 ? 1.0 / diag[m] : 0.0) : 1.0) : 0.0;
}

// ordered per-node sums over slots (plan.cu); what = 1: diag(A)
void slot_sum(const Plan *p, int what, const double *b_e, const int32_t *old_of_new, double *out,
              cudaStream_t s);

// ------------------------------------------------------------ power iteration --
// spectrum.py:64-99.  Ctl reuse: rz = lam (previous quotient), alpha = nav, pq = result,
// k = step, done.
struct PowerEpi {
    const uint8_t *__restrict__ free_int;
    double *__restrict__ av;
    double part[2];
    __device__ __forceinline__ void operator()(int64_t m, double s, double vo) {
        double a = free_int[m] ? s : 0.0;  // spectrum.py:60 out[nd] = 0
        av[m] = a;
        part[0] += vo * a;
        part[1] += a * a;
    }
};

template <int NB, int IDS>
__global__ void EBS_SELL_BOUNDS(NB)
    k_power_matvec(SellView v, Ctl *ctl, double *partials, const double *__restrict__ vin,
                   PowerEpi epi, double tol) {
    if (ctl->done) return;
    sell_sweep<NB, IDS, false>(v, vin, epi);
    double tot[2];
    if (!grid_sum_last<2>(epi.part, partials, &ctl->counter, tot) || threadIdx.x != 0) return;
    const double lam_new = tot[0];
    const double nav = sqrt(tot[1]);
    ctl->k += 1;
    ctl->alpha = nav;
    if (nav == 0.0) {
        ctl->pq = 0.0;
        ctl->done = 1;
        return;
    }
    if (fabs(lam_new - ctl->rz) <= tol * fmax(1.0, fabs(lam_new))) {
        ctl->pq = lam_new;
        ctl->done = 1;
        return;
    }
    ctl->rz = lam_new;
    ctl->pq = lam_new;
}

// v = av / nav (spectrum.py:94); av may alias v (the start vector is scaled in place)
__global__ void k_power_scale(int64_t n, const Ctl *ctl, const double *av, double *v) {
    if (ctl->done && ctl->alpha == 0.0) return;
    const double nav = ctl->alpha;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x)
        v[m] = av[m] / nav;
}

// v = free ? v : 0 and ||v||^2 (start vector, spectrum.py:81-86)
__global__ void k_power_start(int64_t n, const uint8_t *__restrict__ free_int,
                              double *__restrict__ v, double *partials, unsigned int *counter,
                              Ctl *ctl) {
    double part[1] = {0.0};
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        double x = free_int[m] ? v[m] : 0.0;
        v[m] = x;
        part[0] += x * x;
    }
    double tot[1];
    if (grid_sum_last<1>(part, partials, counter, tot) && threadIdx.x == 0) ctl->alpha = sqrt(tot[0]);
}

static void ensure_hist(Plan *p, int64_t n) {
    if (p->hist_cap < n) {
        dfree(p->hist_dev);
        p->hist_dev = dmalloc<double>(2 * n);
        p->hist_cap = n;
    }
}

// --------------------------------------------------- fused single-kernel CG / PCG --
// The whole iteration loop as ONE cooperative persistent kernel (north star: "an
// optional fully fused per-iteration kernel"): per iteration three grid-wide barriers
//   A  q = mask(A p) (SELL sweep), block partials of p.q            | grid.sync
//   B  every block reduces the partials in the same fixed order -> alpha;
//      x += alpha p, r -= alpha q, partials of r.r, r.z (+ err, non-finite count)  | sync
//   C  every block reduces -> the _iterate rules (history, tol, divergence), beta;
//      p = z + beta p                                                  | grid.sync
// No launches or host round trips inside the solve; every block derives the same
// scalars from the same partials, so the loop stays in lockstep.  Arithmetic per node
// is that of k_pcg_update / k_pcg_direction; the dots are reduced over this kernel's
// grid (same results up to rounding, deterministic run to run).
template <int NV>
__device__ __forceinline__ void grid_totals(const double *partials, int G, double (&tot)[NV],
                                            double *smem, double *bc) {
    double w[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < G; b += blockDim.x) acc += __ldcg(&partials[q * G + b]);
        w[q] = acc;
    }
    block_sum<NV>(w, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) bc[q] = w[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) tot[q] = bc[q];
    __syncthreads();
}

// MINB: resident CTAs per SM the register budget is sized for.  Small (latency-bound)
// meshes use 4 (no spills: C1 16.6 us/it vs 26 us/it for three launches); meshes that fill
// the GPU use the SELL kernels' occupancy (6 / 8), at parity with the launch-per-step loop.
template <int NB, int IDS, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_pcg_fused(SellView v, LoopArgs L, int64_t n, int iters, double *__restrict__ x,
                double *__restrict__ r, double *__restrict__ p, double *__restrict__ q,
                const double *__restrict__ dinv, const uint8_t *__restrict__ free_int,
                const double *__restrict__ ref, double *__restrict__ gpart) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sm[4 * 32];
    __shared__ double bc[4];
    Ctl *ctl = L.ctl;
    if (ctl->done) return;  // set by k_pcg_init (tol met at k = 0): uniform over the grid
    const int G = gridDim.x;
    double *pa = gpart, *pb = gpart + G;
    double rz = ctl->rz;
    const double norm0 = ctl->norm0;
    const int64_t stride = (int64_t)G * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    int k = 0, done = 0, diverged = 0;
    while (k < iters) {
        // A: q = mask(A p), p.q
        PcgMatvecEpi me{free_int, q, {0.0}};
        sell_sweep<NB, IDS, false>(v, p, me);
        double a1[1] = {me.part[0]};
        block_sum<1>(a1, sm);
        if (threadIdx.x == 0) pa[blockIdx.x] = a1[0];
        grid.sync();
        double pq[1];
        grid_totals<1>(pa, G, pq, sm, bc);
        const double alpha = pq[0] != 0.0 ? rz / pq[0] : 0.0;
        // B: x, r update, r.r, r.z (+ error, non-finite count)
        double part[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t m = tid; m < n; m += stride) {
            const double xn = x[m] + alpha * p[m];
            const double rn = r[m] - alpha * q[m];
            x[m] = xn;
            r[m] = rn;
            part[0] += rn * rn;
            part[1] += rn * (dinv[m] * rn);
            if (ref) {
                const double d = xn - ref[m];
                part[2] += d * d;
            }
            part[3] += isfinite(xn) ? 0.0 : 1.0;
        }
        block_sum<4>(part, sm);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) pb[i * G + blockIdx.x] = part[i];
        }
        grid.sync();
        double tot[4];
        grid_totals<4>(pb, G, tot, sm, bc);
        // C: the _iterate rules (solvers.py:117-160), identical in every block
        ++k;
        const double nr = sqrt(tot[0]);
        if (tot[3] != 0.0 || !isfinite(nr)) {
            if (leader) {
                L.norms[k] = tot[3] != 0.0 ? INFINITY : nr;
                if (L.errors) L.errors[k] = tot[3] != 0.0 ? INFINITY : sqrt(tot[2]);
            }
            diverged = done = 1;
            break;
        }
        if (leader) {
            L.norms[k] = nr;
            if (L.errors) L.errors[k] = sqrt(tot[2]);
        }
        if (L.has_tol && nr <= L.tol * norm0) {
            done = 1;
            break;
        }
        const double beta = rz != 0.0 ? tot[1] / rz : 0.0;
        rz = tot[1];
        if (k == iters) break;  // the last direction update would be unused
        for (int64_t m = tid; m < n; m += stride) p[m] = dinv[m] * r[m] + beta * p[m];
        grid.sync();
    }
    if (leader) {
        ctl->k = k;
        ctl->n_norms = k + 1;
        ctl->rz = rz;
        ctl->diverged = diverged;
        ctl->done = done;
        ctl->cb_ok = 0;
    }
}

template <int NB, int IDS>
void launch_pcg_fused(Plan *p, const LoopArgs &L, int iters, double *x, double *r, double *pv,
                      double *qv, const double *dinv, const double *ref, cudaStream_t s) {
    constexpr int MINB_BIG = NB == 3 ? EBS_MINB2 : EBS_MINB3;
    const bool small = (p->n_chunks * LANES + 255) / 256 < sm_count() * 4;
    auto kern = small ? k_pcg_fused<NB, IDS, 4> : k_pcg_fused<NB, IDS, MINB_BIG>;
    int per_sm = 0, sms = 0, dev = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int grid = per_sm * sms;  // co-resident by construction (cooperative launch checks it)
    const int64_t work = (p->n_chunks * LANES + 255) / 256;
    if (grid > work) grid = (int)(work > 0 ? work : 1);
    if (grid > RED_MAX_BLOCKS) grid = RED_MAX_BLOCKS;
    SellView v = sell_view(p);
    int64_t n = p->n_n;
    double *gpart = L.partials;  // 5 * RED_MAX_BLOCKS doubles (plan partials)
    const uint8_t *fr = p->free_int;
    void *args[] = {&v, const_cast<LoopArgs *>(&L), &n, &iters, &x, &r, &pv, &qv,
                    const_cast<double **>(&dinv), const_cast<uint8_t **>(&fr),
                    const_cast<double **>(&ref), &gpart};
    CU(cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(256), args, 0, s));
    bump_launches(1);
}

// ------------------------------------------- single-cluster CG / PCG (small meshes) --
// pcg/cg(fused=True) on a mesh whose slot stream fits the shared memory of one thread-
// block cluster (8, else up to 16 CTAs on as many SMs; C1: 4225 nodes, 715 KB of slot
// rows; 4.8 us per iteration vs 11.8 for the cooperative grid kernel): CTA c
// copies the slot rows of its chunks and a full copy of p into its shared memory once,
// then every iteration runs from on-chip memory --
//   A  q = mask(A p) for its own nodes (slot rows and x gathers from shared memory; each
//      thread keeps its node's x, r, p, diag^-1 in registers), p.q block partial
//      broadcast into every CTA's partial array                         | wait mbarrier A
//   B  alpha from the partials summed in rank order (the same in every CTA); x, r
//      update, r.r / r.z / error / non-finite partials broadcast          | wait mbarrier B
//   C  the _iterate rules, beta; p = z + beta p written into every CTA's copy of p
//                                                                         | wait mbarrier C
// The broadcasts are st.async DSMEM stores that complete transaction bytes on the
// receiving CTA's mbarrier, so each CTA waits only for the data it needs -- no
// cluster-wide barrier and fence per phase (C1: 693 -> 621 us per solve in-kernel).
// Reuse is safe without barriers: a CTA sends phase-X data of iteration k+1 only after
// it has received everyone's phase-C data of iteration k, which every CTA sends after
// reading its phase-X data of iteration k.
// -- no global-memory traffic or grid-wide barriers inside the loop.  The row sums are
// sell_node_sum's (same order, same bits); the dots are reduced over the cluster in a
// fixed order (deterministic; equal to the other loops up to rounding).
constexpr int CL_MAX = 16;
constexpr int CL_HIST = 512;  // history entries buffered in shared memory

#ifndef EBS_CLUSTER_MBAR
#define EBS_CLUSTER_MBAR 1  // DSMEM st.async + per-CTA mbarriers instead of cluster barriers
#endif

__device__ __forceinline__ uint32_t cl_mapa(const void *p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(r)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
// 8 B store into another CTA's shared memory, completing 8 tx bytes on its mbarrier
__device__ __forceinline__ void cl_st_async(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void cl_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "CLW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra CLW_%=;\n"
        "}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
        "r"(parity)
        : "memory");
}

// history entries k-cnt+1 .. k (1-based iteration index) from the buffer to global
__device__ __forceinline__ void flush_hist(const LoopArgs &L, const double *hist, int k, int cnt) {
    for (int i = 0; i < cnt; ++i) {
        L.norms[k - cnt + 1 + i] = hist[i];
        if (L.errors) L.errors[k - cnt + 1 + i] = hist[CL_HIST + i];
    }
}

template <int NB, int IDS>
__device__ __forceinline__ double smem_node_sum(const uint8_t *rows, int rowb, int64_t rrel,
                                                int w, int lane, int64_t m, int c_m,
                                                const double *ps, double xo,
                                                const uint8_t *codes, const int4 *tab) {
    double s = 0.0;
    for (int k = 0; k < w; ++k) {
        if (k < c_m) {
            const uint8_t *rp = rows + (rrel + k) * rowb;
            const double *ap = reinterpret_cast<const double *>(rp) + lane;
            double a[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) a[i] = ap[i * LANES];
            int32_t nid[NB - 1];
            int j;
            if constexpr (IDS == IDS_TUPLE) {
                const int4 tp = tab[codes[(rrel + k) * LANES + lane]];
                j = tp.x;
                nid[0] = (int32_t)m + tp.y;
                nid[1] = (int32_t)m + tp.z;
                if constexpr (NB == 4) nid[2] = (int32_t)m + tp.w;
            } else if constexpr (IDS == IDS_DELTA) {
                using W = typename Pack<NB>::W;
                const W wd = reinterpret_cast<const W *>(rp + NB * 256)[lane];
                j = Pack<NB>::j(wd);
#pragma unroll
                for (int t = 0; t < NB - 1; ++t) nid[t] = (int32_t)(m + Pack<NB>::d(wd, t));
            } else {
                const int32_t *ip = reinterpret_cast<const int32_t *>(rp + NB * 256) + lane;
                j = (int)((uint32_t)ip[0] >> J_SHIFT);
#pragma unroll
                for (int t = 0; t < NB - 1; ++t) nid[t] = ip[t * LANES] & ID_MASK;
            }
            double g[NB - 1];
#pragma unroll
            for (int t = 0; t < NB - 1; ++t) g[t] = ps[nid[t]];
            s = s + row_product<NB>(j, a, xo, g);
        }
    }
    return s;
}

template <int NB, int IDS>
__global__ void __launch_bounds__(1024, 1)
    k_pcg_cluster(SellView v, LoopArgs L, int64_t n, int iters, int cpb, int64_t n_rows,
                  double *__restrict__ x, double *__restrict__ r, double *__restrict__ p,
                  const double *__restrict__ dinv, const uint8_t *__restrict__ free_int,
                  const double *__restrict__ ref) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int G = (int)cl.num_blocks();
    const int me = (int)cl.block_rank();
    Ctl *ctl = L.ctl;
    extern __shared__ __align__(16) uint8_t dsm[];
    const int64_t npad = v.n_chunks * LANES;
    double *ps = reinterpret_cast<double *>(dsm);  // full copy of p
    double *pA = ps + npad;                        // [CL_MAX]      p.q partial per rank
    double *pB = pA + CL_MAX;                      // [4 * CL_MAX]  r.r, r.z, err, non-finite
    double *sm = pB + 4 * CL_MAX;                  // [4 * 32]      block_sum scratch
    double *hist = sm + 4 * 32;                    // [2 * CL_HIST] norms / errors, flushed
    int4 *tabs = reinterpret_cast<int4 *>(hist + 2 * CL_HIST);  // [TUPLE_CAP] (IDS_TUPLE)
    uint8_t *rows = reinterpret_cast<uint8_t *>(tabs + TUPLE_CAP);
    __shared__ uint64_t mbar[3];  // A: p.q partials, B: four partials, C: the new p
    if (EBS_CLUSTER_MBAR && threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(&mbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t phase = 0;  // parity bit per barrier
    const int64_t c0 = (int64_t)me * cpb;
    const int64_t c1 = c0 + cpb < v.n_chunks ? c0 + cpb : v.n_chunks;
    const int64_t r0 = c0 < v.n_chunks ? v.rowbase[c0] : n_rows;
    const int64_t r1 = c1 < v.n_chunks ? v.rowbase[c1] : n_rows;
    {  // one-time staging: this CTA's slot rows, all of p
        const int4 *src = reinterpret_cast<const int4 *>(v.slot + r0 * v.rowb);
        int4 *dst = reinterpret_cast<int4 *>(rows);
        const int64_t n16 = (r1 - r0) * v.rowb / 16;
        for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
        for (int64_t i = threadIdx.x; i < npad; i += blockDim.x) ps[i] = i < n ? p[i] : 0.0;
        if constexpr (IDS == IDS_TUPLE) {  // the row codes (32 B per row) and the table
            const int4 *cs = reinterpret_cast<const int4 *>(v.codes + r0 * LANES);
            int4 *cd = reinterpret_cast<int4 *>(rows + (r1 - r0) * v.rowb);
            for (int64_t i = threadIdx.x; i < (r1 - r0) * 2; i += blockDim.x) cd[i] = cs[i];
            for (int i = threadIdx.x; i < TUPLE_CAP; i += blockDim.x) tabs[i] = v.tup[i];
        }
    }
    const uint8_t *codes = rows + (r1 - r0) * v.rowb;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = c0 + wib;
    const int64_t m = c * LANES + lane;
    const bool mine = c < c1 && m < n;
    const int w = c < c1 ? v.width[c] : 0;
    const int c_m = mine ? v.cnt[m] : 0;
    const int64_t rrel = c < c1 ? v.rowbase[c] - r0 : 0;
    double xm = 0.0, rm = 0.0, pm = 0.0, dm = 0.0, refm = 0.0;
    bool fm = false;
    if (mine) {
        xm = x[m], rm = r[m], pm = p[m], dm = dinv[m], fm = free_int[m] != 0;
        if (ref) refm = ref[m];
    }
    double rz = ctl->rz;
    const double norm0 = ctl->norm0;
    const bool leader = me == 0 && threadIdx.x == 0;
    int k = 0, done = ctl->done, diverged = 0;
    cl.sync();  // staging complete everywhere (ps is read by the gathers)
    while (!done && k < iters) {
        // A: q = mask(A p), p.q
        double qm = 0.0;
        {
            const double s = smem_node_sum<NB, IDS>(rows, v.rowb, rrel, w, lane, m, c_m, ps, pm,
                                                    codes, tabs);
            if (mine) qm = fm ? s : 0.0;
        }
        double a1[1] = {pm * qm};
        block_sum<1>(a1, sm);
        if (EBS_CLUSTER_MBAR) {
            if (threadIdx.x == 0) mbar_expect_tx(&mbar[0], 8u * G);
            if (wib == 0) {  // block total -> slot `me` of every CTA's pA, signalling its barrier
                const double tv = __shfl_sync(0xffffffffu, a1[0], 0);
                if (lane < G) cl_st_async(cl_mapa(pA + me, lane), tv, cl_mapa(&mbar[0], lane));
            }
            cl_wait(&mbar[0], phase & 1u);
            phase ^= 1u;
        } else {
            if (wib == 0) {  // block total (lane 0 of warp 0) -> slot `me` of every CTA's pA
                const double tv = __shfl_sync(0xffffffffu, a1[0], 0);
                if (lane < G) *cl.map_shared_rank(pA + me, lane) = tv;
            }
            cl.sync();
        }
        double pq = 0.0;
        for (int t = 0; t < G; ++t) pq += pA[t];
        const double alpha = pq != 0.0 ? rz / pq : 0.0;
        // B: x, r update, r.r, r.z (+ error, non-finite count)
        double part[4] = {0.0, 0.0, 0.0, 0.0};
        if (mine) {
            xm = xm + alpha * pm;
            rm = rm - alpha * qm;
            part[0] = rm * rm;
            part[1] = rm * (dm * rm);
            if (ref) {
                const double d = xm - refm;
                part[2] = d * d;
            }
            part[3] = isfinite(xm) ? 0.0 : 1.0;
        }
        block_sum<4>(part, sm);
        if (EBS_CLUSTER_MBAR) {
            if (threadIdx.x == 0) mbar_expect_tx(&mbar[1], 32u * G);
            if (wib == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double tv = __shfl_sync(0xffffffffu, part[q], 0);
                    if (lane < G)
                        cl_st_async(cl_mapa(pB + q * CL_MAX + me, lane), tv, cl_mapa(&mbar[1], lane));
                }
            }
            cl_wait(&mbar[1], (phase >> 1) & 1u);
            phase ^= 2u;
        } else {
            if (wib == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double tv = __shfl_sync(0xffffffffu, part[q], 0);
                    if (lane < G) *cl.map_shared_rank(pB + q * CL_MAX + me, lane) = tv;
                }
            }
            cl.sync();
        }
        double tot[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t = 0; t < G; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q) tot[q] += pB[q * CL_MAX + t];
        // C: the _iterate rules (solvers.py:117-160), identical in every CTA
        ++k;
        const double nr = sqrt(tot[0]);
        // history entries go to a shared-memory buffer, flushed when full and at the end:
        // a global store before a cluster barrier makes its release fence wait for it
        const bool bad = tot[3] != 0.0 || !isfinite(nr);
        if (leader) {
            const int h = (k - 1) % CL_HIST;
            hist[h] = bad && tot[3] != 0.0 ? INFINITY : nr;
            hist[CL_HIST + h] = bad && tot[3] != 0.0 ? INFINITY : sqrt(tot[2]);
            if (h == CL_HIST - 1) flush_hist(L, hist, k, h + 1);
        }
        if (bad) {
            diverged = done = 1;
            break;
        }
        if (L.has_tol && nr <= L.tol * norm0) {
            done = 1;
            break;
        }
        const double beta = rz != 0.0 ? tot[1] / rz : 0.0;
        rz = tot[1];
        if (k == iters) break;  // the last direction update would be unused
        if (mine) pm = dm * rm + beta * pm;
        if (EBS_CLUSTER_MBAR) {  // every node's p into every CTA's copy: 8 n bytes per CTA
            if (threadIdx.x == 0) mbar_expect_tx(&mbar[2], (uint32_t)(8 * n));
            if (mine)
                for (int t = 0; t < G; ++t) cl_st_async(cl_mapa(ps + m, t), pm, cl_mapa(&mbar[2], t));
            cl_wait(&mbar[2], (phase >> 2) & 1u);
            phase ^= 4u;
        } else {
            if (mine)
                for (int t = 0; t < G; ++t) *cl.map_shared_rank(ps + m, t) = pm;
            cl.sync();
        }
    }
    if (mine) {
        x[m] = xm;
        r[m] = rm;
        p[m] = pm;
    }
    if (leader) {
        if (k > 0 && (k - 1) % CL_HIST != CL_HIST - 1) flush_hist(L, hist, k, (k - 1) % CL_HIST + 1);
        ctl->k = k;
        ctl->n_norms = k + 1;
        ctl->rz = rz;
        ctl->diverged = diverged;
        ctl->done = done;
        ctl->cb_ok = 0;
    }
    cl.sync();  // no CTA exits while others may still write into its shared memory
}

#ifndef EBS_PCG_CLUSTER
#define EBS_PCG_CLUSTER 1
#endif

// Launch k_pcg_cluster when the mesh fits one cluster; false: use the cooperative kernel.
template <int NB, int IDS>
bool launch_pcg_cluster(Plan *p, const LoopArgs &L, int iters, double *x, double *r, double *pv,
                        const double *dinv, const double *ref, cudaStream_t s) {
    if (!EBS_PCG_CLUSTER || getenv("EBS_NO_CLUSTER")) return false;
    if constexpr (IDS != IDS_DELTA && IDS != IDS_ABS && IDS != IDS_TUPLE) {
        return false;
    } else {
        auto kern = k_pcg_cluster<NB, IDS>;
        if (p->cl_state == 0) {  // choose the cluster once per plan
            p->cl_state = -1;
            const int64_t nch = p->n_chunks;
            if (nch < 1 || nch > (int64_t)CL_MAX * 32) return false;
            std::vector<int32_t> rb(nch);
            CU(cudaMemcpyAsync(rb.data(), p->rowbase, sizeof(int32_t) * nch, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            const char *ge = getenv("EBS_CLUSTER_MAX");
            const int gmax = ge ? atoi(ge) : CL_MAX;
            for (int G : {8, CL_MAX, 4, 2}) {  // 8 first: C1 5.3 vs 5.6 us/it at 16
                if (G > gmax) continue;
                const int cpb = (int)((nch + G - 1) / G);
                if (cpb * 32 > 1024) continue;
                int64_t max_rows = 0;
                for (int c = 0; c < G; ++c) {
                    const int64_t a = (int64_t)c * cpb, b = a + cpb < nch ? a + cpb : nch;
                    if (a >= nch) break;
                    const int64_t ra = rb[a], rbnd = b < nch ? rb[b] : p->n_rows;
                    max_rows = rbnd - ra > max_rows ? rbnd - ra : max_rows;
                }
                const size_t smem = sizeof(double) * (nch * 32 + 5 * CL_MAX + 4 * 32 + 2 * CL_HIST) +
                                    sizeof(int4) * TUPLE_CAP +
                                    (size_t)max_rows * (p->rowb + (IDS == IDS_TUPLE ? LANES : 0));
                if (smem > 227 * 1024) continue;
                if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
                    (G > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
                    cudaGetLastError();
                    continue;
                }
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(G);
                cfg.blockDim = dim3(cpb * 32);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = G;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                int clusters = 0;
                if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters < 1) {
                    cudaGetLastError();
                    continue;
                }
                p->cl_state = 1, p->cl_G = G, p->cl_cpb = cpb, p->cl_smem = smem;
                break;
            }
        }
        if (p->cl_state != 1) return false;
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->cl_smem));
        if (p->cl_G > 8) CU(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p->cl_G);
        cfg.blockDim = dim3(p->cl_cpb * 32);
        cfg.dynamicSmemBytes = p->cl_smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = p->cl_G;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        SellView v = sell_view(p);
        int64_t n = p->n_n, n_rows = p->n_rows;
        const int cpb = p->cl_cpb;
        CU(cudaLaunchKernelEx(&cfg, kern, v, L, n, iters, cpb, n_rows, x, r, pv, dinv,
                              (const uint8_t *)p->free_int, ref));
        bump_launches(1);
        return true;
    }
}

}  // namespace ebs

using namespace ebs;


#ifndef EBS_SOLVE_GRAPH
#define EBS_SOLVE_GRAPH 1  // replay 32-iteration batches from a captured CUDA graph
#endif

// Runs iterations [k0, iters) of a device-controlled solver loop in batches of `batch`:
// `body(st)` enqueues one iteration on stream st (every launch identical -- the
// iteration index and stop state live in the device control block).  Full batches after
// the first are replayed from a CUDA graph captured on the plan's capture stream; one
// batch stays queued ahead of the host's look at the stop flag (no per-batch bubble).
// Returns the first iteration index not enqueued; *done = the device stopped the loop.
template <class Body>
static int run_batches(Plan *p, int k0, int iters, int batch, cudaStream_t s, Body body,
                       bool *done) {
    int k = k0;
    *done = false;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    const bool use_graph = EBS_SOLVE_GRAPH && iters - k0 >= 3 * batch;
    if (!p->ring_ev[0]) {
        for (auto &e : p->ring_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    int pending = -1;  // ring slot of the batch whose stop flag has not been read yet
    int slot = 0;
    int64_t per_batch = 0;
    try {
        while (k < iters && !*done) {
            const int kend = k + batch < iters ? k + batch : iters;
            if (use_graph && kend - k == batch && k > k0) {
                if (!exec) {
                    if (!p->cap_stream)
                        CU(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
                    const int64_t c0 = bump_launches(0);
                    CU(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
                    try {
                        for (int u = 0; u < batch; ++u) body(p->cap_stream);
                    } catch (...) {
                        cudaStreamEndCapture(p->cap_stream, &graph);
                        throw;
                    }
                    CU(cudaStreamEndCapture(p->cap_stream, &graph));
                    CU(cudaGraphInstantiate(&exec, graph, 0));
                    per_batch = bump_launches(0) - c0;  // captured, not run: count at replay
                    bump_launches(-per_batch);
                }
                CU(cudaGraphLaunch(exec, s));
                bump_launches(per_batch);
            } else {
                for (int u = k; u < kend; ++u) body(s);
            }
            k = kend;
            CU(cudaMemcpyAsync(p->ctl_host + 1 + slot, p->ctl, sizeof(Ctl),
                               cudaMemcpyDeviceToHost, s));
            CU(cudaEventRecord(p->ring_ev[slot], s));
            if (pending >= 0) {
                CU(cudaEventSynchronize(p->ring_ev[pending]));
                *done = p->ctl_host[1 + pending].done != 0;
            }
            pending = slot;
            slot ^= 1;
        }
        if (pending >= 0 && !*done) {
            CU(cudaEventSynchronize(p->ring_ev[pending]));
            *done = p->ctl_host[1 + pending].done != 0;
        }
    } catch (...) {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        cudaStreamSynchronize(s);
        throw;
    }
    if (exec) {
        CU(cudaStreamSynchronize(s));
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
    }
    return k;
}

extern "C" {

int ebs_solve(ebs_plan_t plan, const ebs_solve_params *P, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && P, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    EBS_REQUIRE(P->iters >= 0, "iteration count must be nonnegative, got %d", P->iters);
    EBS_REQUIRE(P->method >= EBS_RICHARDSON && P->method <= EBS_CHEB3, "bad method %d", P->method);
    EBS_REQUIRE(P->method != EBS_CHEB2 || P->coef_a || P->iters == 0, "CHEB2 needs coef_a");
    EBS_REQUIRE(P->method != EBS_CHEB3 || ((P->coef_a && P->coef_b) || P->iters == 0),
                "CHEB3 needs coef_a and coef_b");
    EBS_REQUIRE(p->has_A && p->has_be, "solver needs an operator loaded with b_e");
    EBS_REQUIRE(P->x0 && P->x && P->norms && P->n_norms && P->diverged, "null argument");
    EBS_REQUIRE(!P->reference || P->errors, "errors buffer required with reference");
    EBS_REQUIRE(!P->callback || (P->cb_x && P->cb_r), "callback needs cb_x and cb_r");
    cudaStream_t s = S(stream);
    const int64_t n = p->n_n;
    const int iters = P->iters;
    const int nb = p->nb;
    // history: norms [0, iters+2), errors [iters+2, 2(iters+2)), then 2*iters coefficients
    ensure_hist(p, 2 * ((int64_t)iters + 2) + (int64_t)iters);
    double *xa = plan_vec(p, 1), *xb = plan_vec(p, 2), *r_int = plan_vec(p, 3);
    double *dinv = plan_vec(p, 4), *ref_int = nullptr;
    CU(cudaMemsetAsync(p->ctl, 0, sizeof(Ctl), s));
    CU(cudaMemsetAsync(p->hist_dev, 0, sizeof(double) * 2 * ((int64_t)iters + 2), s));
    to_internal(p, P->x0, xa, &p->ctl->x0_nonfinite, s);
    if (P->callback) {  // the reference raises before its first callback
        CU(cudaMemcpyAsync(p->ctl_host, p->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (p->ctl_host->x0_nonfinite) {
            set_error("x contains non-finite entries");
            return EBS_ENONFINITE;
        }
    }
    if (P->reference) {
        ref_int = plan_vec(p, 7);
        to_internal(p, P->reference, ref_int, nullptr, s);
    }
    LoopArgs L{p->ctl, p->hist_dev, P->reference ? p->hist_dev + iters + 2 : nullptr,
               p->partials, P->has_tol, P->tol, P->omega};
    SellView v = sell_view(p);
    const int vgrid = grid_for(n, 256, RED_MAX_BLOCKS);
    const int ugrid = EBS_UPD_PERSIST
                          ? persistent_grid((const void *)k_pcg_update, 256, (n + 255) / 256, 0)
                          : vgrid;
    const bool cb = P->callback != nullptr;
    const int batch = cb ? 1 : 32;
    bool aborted = false;

    auto read_ctl = [&]() {
        CU(cudaMemcpyAsync(p->ctl_host, p->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    };
    auto do_callback = [&](const double *x_int_k, int k) {
        to_user(p, x_int_k, P->cb_x, s);
        to_user(p, r_int, P->cb_r, s);
        CU(cudaStreamSynchronize(s));
        if (P->callback(P->user, k) != 0) aborted = true;
    };

    const bool stationary = P->method == EBS_RICHARDSON || P->method == EBS_JACOBI ||
                            P->method == EBS_CHEB2 || P->method == EBS_CHEB3;
    if (n > 0 && stationary) {
        const double *dv = nullptr;
        double *coef_a = nullptr, *coef_b = nullptr, *pbuf = nullptr;
        if ((P->method == EBS_CHEB2 || P->method == EBS_CHEB3) && iters > 0) {
            // coefficient tables live behind the history on the device
            coef_a = p->hist_dev + 2 * ((int64_t)iters + 2);
            coef_b = coef_a + iters;
            CU(cudaMemcpyAsync(coef_a, P->coef_a, sizeof(double) * iters, cudaMemcpyHostToDevice, s));
            if (P->method == EBS_CHEB3) {
                CU(cudaMemcpyAsync(coef_b, P->coef_b, sizeof(double) * iters,
                                   cudaMemcpyHostToDevice, s));
                pbuf = plan_vec(p, 6);
            }
        }
        if (P->method == EBS_JACOBI) {
            double *diag = plan_vec(p, 5);
            slot_sum(p, 1, nullptr, nullptr, diag, s);
            k_dinv<<<grid_for(n, 256), 256, 0, s>>>(n, diag, p->free_int, dinv);
            LAUNCHED();
            dv = dinv;
        }
        const bool exact = P->exact != 0;
        double *rcb = (cb || P->r_out) ? r_int : nullptr;
        auto step = [&](int final_step, cudaStream_t st) {
            if (ref_int) {
                k_err_norm<<<vgrid, 256, 0, st>>>(n, L, xa, xb, ref_int);
                LAUNCHED();
            }
            JacArgs A{p->b_int, p->free_int, dv, ref_int, rcb, xa, xb, pbuf, coef_a, coef_b,
                      final_step};
            const int kind = P->method == EBS_JACOBI ? JK_JACOBI
                                                     : (P->method == EBS_CHEB3 ? JK_CHEB3 : JK_PLAIN);
#define EBS_JAC(NB_, PK_, EX_, KD_)                                                         \
    {                                                                                       \
        auto kern = k_jacobi_step<NB_, PK_, EX_, KD_>;                                      \
        const SellLaunch SL = sell_launch((const void *)kern, NB_, p->rowb, p->n_chunks);   \
        kern<<<SL.grid, SL.block, SL.smem, st>>>(v, L, A);                                  \
    }
#define EBS_JAC_K(NB_, PK_, EX_)                                                            \
    {                                                                                       \
        if (kind == JK_JACOBI) EBS_JAC(NB_, PK_, EX_, JK_JACOBI)                            \
        else if (kind == JK_CHEB3) EBS_JAC(NB_, PK_, EX_, JK_CHEB3)                         \
        else EBS_JAC(NB_, PK_, EX_, JK_PLAIN)                                               \
    }
#define EBS_JAC_T(NB_, IDS_) { if (exact) EBS_JAC_K(NB_, IDS_, true) else EBS_JAC_K(NB_, IDS_, false) }
            EBS_SELL_DISPATCH(p, EBS_JAC_T);
#undef EBS_JAC_T
#undef EBS_JAC_K
#undef EBS_JAC
            LAUNCHED();
        };
        int k = 0;
        bool done = false;
        if (!cb) {
            k = run_batches(p, 0, iters, batch, s, [&](cudaStream_t st) { step(0, st); }, &done);
            read_ctl();  // final_buf below
        }
        while (k < iters && !done && !aborted) {
            int kend = k + batch < iters ? k + batch : iters;
            for (; k < kend; ++k) step(0, s);
            read_ctl();
            done = p->ctl_host->done != 0;
            if (cb && p->ctl_host->cb_ok) {
                int kk = p->ctl_host->n_norms - 1;
                if (p->ctl_host->nonfinite) kk = p->ctl_host->n_norms - 2;
                do_callback(((kk & 1) ? xb : xa), kk);
            }
        }
        if (!done && !aborted) {
            step(1, s);
            read_ctl();
            if (cb) do_callback(((iters & 1) ? xb : xa), iters);
        }
        const double *xf = (p->ctl_host->final_buf & 1) ? xb : xa;
        to_user(p, xf, P->x, s);
    } else if (n > 0) {
        // CG / PCG
        double *pv = plan_vec(p, 5), *qv = plan_vec(p, 6);
        double *diag = nullptr;
        if (P->method == EBS_PCG) {
            diag = qv;  // scratch before the loop
            slot_sum(p, 1, nullptr, nullptr, diag, s);
        }
        k_dinv<<<grid_for(n, 256), 256, 0, s>>>(n, diag, p->free_int, dinv);
        LAUNCHED();
        {
            PcgInitEpi ie{p->b_int, p->free_int, dinv, ref_int, r_int, pv, {0.0, 0.0, 0.0}};
#define EBS_INIT(NB_, PK_)                                                                  \
    {                                                                                       \
        auto kern = k_pcg_init<NB_, PK_>;                                                   \
        const SellLaunch SL = sell_launch((const void *)kern, NB_, p->rowb, p->n_chunks);   \
        kern<<<SL.grid, SL.block, SL.smem, s>>>(v, L, xa, ie);                              \
    }
            EBS_SELL_DISPATCH(p, EBS_INIT);
#undef EBS_INIT
            LAUNCHED();
        }
        if (cb) {
            read_ctl();
            do_callback(xa, 0);
        }
        auto iteration = [&](cudaStream_t st) {
            {
                PcgMatvecEpi me{p->free_int, qv, {0.0}};
#define EBS_MV(NB_, PK_)                                                                    \
    {                                                                                       \
        auto kern = k_pcg_matvec<NB_, PK_>;                                                 \
        const SellLaunch SL = sell_launch((const void *)kern, NB_, p->rowb, p->n_chunks);   \
        kern<<<SL.grid, SL.block, SL.smem, st>>>(v, L, pv, me);                             \
    }
                EBS_SELL_DISPATCH(p, EBS_MV);
#undef EBS_MV
            }
            LAUNCHED();
            k_pcg_update<<<ugrid, 256, 0, st>>>(n, L, xa, r_int, pv, qv, dinv, ref_int);
            LAUNCHED();
            k_pcg_direction<<<grid_for(n, 256), 256, 0, st>>>(n, p->ctl, pv, r_int, dinv);
            LAUNCHED();
        };
        int k = 0;
        bool done = false;
        if (P->fused && !cb && iters > 0) {  // the whole loop as one cooperative kernel
#define EBS_FUSED(NB_, PK_)                                                                  \
    {                                                                                        \
        if (!launch_pcg_cluster<NB_, PK_>(p, L, iters, xa, r_int, pv, dinv, ref_int, s))     \
            launch_pcg_fused<NB_, PK_>(p, L, iters, xa, r_int, pv, qv, dinv, ref_int, s);    \
    }
            EBS_SELL_DISPATCH(p, EBS_FUSED);
#undef EBS_FUSED
            k = iters;
        } else if (!cb) {
            k = run_batches(p, 0, iters, batch, s, iteration, &done);
        }
        while (k < iters && !done && !aborted) {
            int kend = k + batch < iters ? k + batch : iters;
            for (; k < kend; ++k) iteration(s);
            read_ctl();
            done = p->ctl_host->done != 0;
            if (cb && p->ctl_host->cb_ok) do_callback(xa, p->ctl_host->n_norms - 1);
        }
        read_ctl();
        to_user(p, xa, P->x, s);
    } else {
        read_ctl();
    }
    if (P->r_out && n > 0) to_user(p, r_int, P->r_out, s);
    read_ctl();
    const int nn = n > 0 ? p->ctl_host->n_norms : 0;
    *P->n_norms = nn;
    *P->diverged = p->ctl_host->diverged;
    if (nn > 0) {
        CU(cudaMemcpyAsync(P->norms, p->hist_dev, sizeof(double) * nn, cudaMemcpyDeviceToHost, s));
        if (P->reference)
            CU(cudaMemcpyAsync(P->errors, p->hist_dev + iters + 2, sizeof(double) * nn,
                               cudaMemcpyDeviceToHost, s));
    }
    CU(cudaStreamSynchronize(s));
    if (p->ctl_host->x0_nonfinite) {  // _iterate's first residual() raises (operators.py:90)
        set_error("x contains non-finite entries");
        return EBS_ENONFINITE;
    }
    if (aborted) {
        set_error("solve stopped by callback");
        return EBS_ECALLBACK;
    }
    EBS_CATCH
}

int ebs_power_iteration(ebs_plan_t plan, const double *v0, int iters, double tol, double *lam,
                        int *its, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && v0 && lam && its, "null argument");
    EBS_REQUIRE(iters >= 1, "need at least one iteration, got %d", iters);
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    cudaStream_t s = S(stream);
    const int64_t n = p->n_n;
    double *v = plan_vec(p, 1), *av = plan_vec(p, 2);
    CU(cudaMemsetAsync(p->ctl, 0, sizeof(Ctl), s));
    to_internal(p, v0, v, nullptr, s);
    k_power_start<<<grid_for(n, 256, RED_MAX_BLOCKS), 256, 0, s>>>(n, p->free_int, v, p->partials,
                                                                  &p->ctl->counter, p->ctl);
    LAUNCHED();
    CU(cudaMemcpyAsync(p->ctl_host, p->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const double nv = p->ctl_host->alpha;
    if (nv == 0.0) {
        set_error("start vector vanished after masking (no free nodes?)");
        return EBS_EINVAL;
    }
    // v /= ||v||: reuse the scale kernel with ctl->alpha = ||v||, done = 0
    k_power_scale<<<grid_for(n, 256), 256, 0, s>>>(n, p->ctl, v, v);
    LAUNCHED();
    CU(cudaMemsetAsync(p->ctl, 0, sizeof(Ctl), s));
    SellView sv = sell_view(p);
    int k = 0;
    while (k < iters) {
        int kend = k + 32 < iters ? k + 32 : iters;
        for (; k < kend; ++k) {
            PowerEpi epi{p->free_int, av, {0.0, 0.0}};
#define EBS_PW(NB_, PK_)                                                                    \
    {                                                                                       \
        auto kern = k_power_matvec<NB_, PK_>;                                               \
        const SellLaunch SL = sell_launch((const void *)kern, NB_, p->rowb, p->n_chunks);   \
        kern<<<SL.grid, SL.block, SL.smem, s>>>(sv, p->ctl, p->partials, v, epi, tol);      \
    }
            EBS_SELL_DISPATCH(p, EBS_PW);
#undef EBS_PW
            LAUNCHED();
            k_power_scale<<<grid_for(n, 256), 256, 0, s>>>(n, p->ctl, av, v);
            LAUNCHED();
        }
        CU(cudaMemcpyAsync(p->ctl_host, p->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (p->ctl_host->done) break;
    }
    CU(cudaMemcpyAsync(p->ctl_host, p->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *lam = p->ctl_host->pq;
    *its = p->ctl_host->k;
    EBS_CATCH
}

}  // extern "C"

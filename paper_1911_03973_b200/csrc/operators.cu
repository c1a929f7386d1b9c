// operators.cu -- residual / matvec entry points (caller numbering in and out).
//
//   ebs_residual  <- operators.py:72-111 residual (+ operators.py:114-118 mask)
//   ebs_matvec    <- spectrum.py:54-61 _apply_masked
//
// Each call is two launches: a gather of x into the plan's internal numbering (with the
// finiteness check of operators.py:90 fused in), then the SELL kernel, whose epilogue
// scatters straight into the caller's numbering.
#include "sell.cuh"

namespace ebs {

__global__ void k_to_internal(int64_t n, const int32_t *__restrict__ old_of_new,
                              const double *__restrict__ x_user, double *__restrict__ x_int,
                              int32_t *nonfinite) {
    bool bad = false;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        double v = x_user[old_of_new[m]];
        bad |= !isfinite(v);
        x_int[m] = v;
    }
    if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(nonfinite, 1);
}

__global__ void k_to_user(int64_t n, const int32_t *__restrict__ old_of_new,
                          const double *__restrict__ v_int, double *__restrict__ v_user) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x)
        v_user[old_of_new[m]] = v_int[m];
}

// Caller-order output of a permuted numbering is one random 8 B store per node: the
// L1tex pipe spends ~2 cycles on each distinct line of a warp's store (ncu: C2 MODE 1
// 161 us vs 131 us with internal-order output).  A fire-and-forget red.add (REDG) into a
// vector pre-filled with -0.0 costs less per lane and is bit-exact: every caller node
// receives exactly one value s, and -0.0 + s == s for every s (IEEE round-to-nearest,
// including s = +0.0 and s = -0.0).  C2: SELL pass 161 -> 150 us.
#ifndef EBS_OUT_RED
#define EBS_OUT_RED 1
#endif

// MODE 0: y = A x   1: r = b - A x (pre-assembled b)   2: r = sum(b_e - A_e x_e) exact
struct OpEpi {
    int mode;
    const double *__restrict__ b_int;
    const uint8_t *__restrict__ free_int;
    const int32_t *__restrict__ old_of_new;
    double *__restrict__ out;
    double *__restrict__ s_raw;  // nullable: the node values again, internal order (halo)
    int red;                     // out[old_of_new[m]] += s into a -0.0-filled vector
    __device__ __forceinline__ void operator()(int64_t m, double s, double) {
        if (mode == 1) s = b_int[m] - s;
        if (free_int && !free_int[m]) s = 0.0;
        if (s_raw) s_raw[m] = s;
        if (old_of_new) {
            if (red) atomicAdd(out + old_of_new[m], s);
            else out[old_of_new[m]] = s;
        } else {
            out[m] = s;
        }
    }
};

template <int NB, int IDS, int MODE>
__global__ void EBS_SELL_BOUNDS(NB)
    k_sell_op(SellView v, const double *__restrict__ x, OpEpi epi) {
    sell_sweep<NB, IDS, MODE == 2>(v, x, epi);
}

template <int NB, int IDS, int MODE>
void launch_sell_op_t(const Plan *p, const double *x_int, const OpEpi &epi, cudaStream_t s,
                      const int32_t *chunks = nullptr, int64_t n_list = -1) {
    auto kern = k_sell_op<NB, IDS, MODE>;
    const SellView v = sell_view(p, chunks, n_list);
    const SellLaunch SL = sell_launch((const void *)kern, NB, p->rowb, v.nlist);
    kern<<<SL.grid, SL.block, SL.smem, s>>>(v, x_int, epi);
    LAUNCHED();
}

template <int MODE>
void launch_sell_op(const Plan *p, const double *x_int, const uint8_t *free_int,
                    const int32_t *old_of_new, double *out, cudaStream_t s,
                    double *s_raw = nullptr, const int32_t *chunks = nullptr,
                    int64_t n_list = -1, int red = 0) {
    if (p->n_n == 0 || n_list == 0) return;
    OpEpi epi{MODE, p->b_int, free_int, old_of_new, out, s_raw, red};
#define EBS_OP(NB_, IDS_) { launch_sell_op_t<NB_, IDS_, MODE>(p, x_int, epi, s, chunks, n_list); }
    EBS_SELL_DISPATCH(p, EBS_OP);
#undef EBS_OP
}

// scatter orientation: coalesced read of x in caller order, 8 B writes into the
// L2-resident internal vector (writes do not stall the issuing warp)
__global__ void k_to_internal_scatter(int64_t n, const int32_t *__restrict__ new_of_old,
                                      const double *__restrict__ x_user,
                                      double *__restrict__ x_int, int32_t *nonfinite) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = x_user[i];
        bad |= !isfinite(v);
        x_int[new_of_old[i]] = v;
    }
    if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(nonfinite, 1);
}

// gather orientation with 8 independent index->value chains per thread (memory-level
// parallelism for the random 8 B reads)
constexpr int PERM_ILP = 8;
#ifndef EBS_PERM_PF
#define EBS_PERM_PF 0  // 0 plain gathers, 1 L2::256B gather hint, 2 bulk L2 prefetch of x first
#endif

__device__ __forceinline__ double ld_x_perm(const double *p) {
#if EBS_PERM_PF == 1
    double v;
    asm volatile("ld.global.nc.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

__global__ void __launch_bounds__(256)
    k_to_internal_ilp(int64_t n, const int32_t *__restrict__ old_of_new,
                      const double *__restrict__ x_user, double *__restrict__ x_int,
                      int32_t *nonfinite, double *__restrict__ negzero) {
    bool bad = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#if EBS_PERM_PF == 2
    {   // stream this block's slice of x into L2 at sequential DRAM efficiency; the random
        // gathers below then mostly hit L2 (a hint only: correctness never depends on it)
        const int64_t bytes = n * 8;
        const int64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 4095) & ~int64_t(4095);
        const int64_t lo = (int64_t)blockIdx.x * per;
        const int64_t hi = lo + per < bytes ? lo + per : bytes;
        for (int64_t o = lo + (int64_t)threadIdx.x * 4096; o < hi;
             o += (int64_t)blockDim.x * 4096) {
            const uint32_t sz = (uint32_t)(bytes - o < 4096 ? bytes - o : 4096) & ~15u;
            if (sz)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                             :: "l"((const char *)x_user + o), "r"(sz) : "memory");
        }
    }
#endif
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n;
         base += stride * PERM_ILP) {
        int32_t idx[PERM_ILP];
        double v[PERM_ILP];
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t m = base + u * stride;
            idx[u] = m < n ? __ldcs(old_of_new + m) : 0;
        }
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t m = base + u * stride;
            v[u] = m < n ? ld_x_perm(x_user + idx[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t m = base + u * stride;
            if (m < n) {
                bad |= !isfinite(v[u]);
                x_int[m] = v[u];
                if (negzero) negzero[m] = -0.0;  // the output of a following red pass
            }
        }
    }
    if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(nonfinite, 1);
}

#ifndef EBS_TO_INTERNAL_SCATTER
#define EBS_TO_INTERNAL_SCATTER 2  // 0 gather, 1 scatter, 2 gather with ILP
#endif

#ifndef EBS_PERM2
// 1: caller <-> internal permutations through the two-pass shared-memory schedule of
// perm.cu (every global access coalesced).  Measured slower at C2 (2 passes 44 us vs the
// direct gather's 33 us; profiles/README.md), so opt-in.
#define EBS_PERM2 0
#endif

// out[0..n) = -0.0 with 16 B stores (scalar head / tail for an unaligned or odd range)
__global__ void k_fill_negzero(int64_t n, double *__restrict__ out) {
    const int64_t head = (reinterpret_cast<uintptr_t>(out) & 15) ? 1 : 0;
    const int64_t n2 = n > head ? (n - head) / 2 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (head && n > 0) out[0] = -0.0;
        if (n > head && ((n - head) & 1)) out[n - 1] = -0.0;
    }
    double2 *o2 = reinterpret_cast<double2 *>(out + head);
    const double2 v = make_double2(-0.0, -0.0);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
         i += (int64_t)gridDim.x * blockDim.x)
        o2[i] = v;
}

#ifndef EBS_FILL_MODE
// -0.0 pre-fill of the red-mode output: 0 fused into the x permutation, 1 separate kernel
// after it, 2 before it.  Measured at C2: 1 best (23.8 GDoF/s; 0: 23.4-23.7 -- the extra
// stores slow the latency-bound gather; 2: 22.6-22.9)
#define EBS_FILL_MODE 1
#endif

static void fill_negzero(int64_t n, double *out, cudaStream_t s) {
    if (n == 0) return;
    k_fill_negzero<<<grid_for((n + 1) / 2, 256, 148 * 8), 256, 0, s>>>(n, out);
    LAUNCHED();
}

// x_user (caller numbering) -> x_int; negzero (nullable, n_n doubles) is set to -0.0 in
// the same pass (the output vector of a following red-mode SELL pass)
void to_internal(const Plan *p, const double *x_user, double *x_int, int32_t *nonfinite,
                 cudaStream_t s, double *negzero) {
    if (p->n_n == 0) return;
    if (negzero && (EBS_PERM2 || EBS_TO_INTERNAL_SCATTER != 2)) {
        fill_negzero(p->n_n, negzero, s);
        negzero = nullptr;
    }
    if (EBS_PERM2) {
        Plan *pm = const_cast<Plan *>(p);
        if (const Perm2 *P = perm_get(pm, 0, s)) {
            perm_apply(pm, P, x_user, x_int, nonfinite, s);
            return;
        }
    }
    if (EBS_TO_INTERNAL_SCATTER == 2)
        k_to_internal_ilp<<<grid_for((p->n_n + PERM_ILP - 1) / PERM_ILP, 256, 148 * 8), 256, 0,
                            s>>>(p->n_n, p->old_of_new, x_user, x_int, nonfinite, negzero);
    else if (EBS_TO_INTERNAL_SCATTER == 1)
        k_to_internal_scatter<<<grid_for(p->n_n, 256, 148 * 32), 256, 0, s>>>(
            p->n_n, p->new_of_old, x_user, x_int, nonfinite);
    else
        k_to_internal<<<grid_for(p->n_n, 256, 148 * 32), 256, 0, s>>>(p->n_n, p->old_of_new,
                                                                      x_user, x_int, nonfinite);
    LAUNCHED();
}

// out_user[n] = v_int[new_of_old[n]]: coalesced writes, random reads of an L2-resident
// internal vector (ILP-8)
__global__ void __launch_bounds__(256)
    k_from_internal_ilp(int64_t n, const int32_t *__restrict__ new_of_old,
                        const double *__restrict__ v_int, double *__restrict__ v_user) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < n;
         base += stride * PERM_ILP) {
        int32_t idx[PERM_ILP];
        double v[PERM_ILP];
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t i = base + u * stride;
            idx[u] = i < n ? __ldcs(new_of_old + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t i = base + u * stride;
            v[u] = i < n ? v_int[idx[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t i = base + u * stride;
            if (i < n) v_user[i] = v[u];
        }
    }
}

void to_user(const Plan *p, const double *v_int, double *v_user, cudaStream_t s) {
    if (p->n_n == 0) return;
    if (EBS_PERM2) {
        Plan *pm = const_cast<Plan *>(p);
        if (const Perm2 *P = perm_get(pm, 1, s)) {
            perm_apply(pm, P, v_int, v_user, nullptr, s);
            return;
        }
    }
    // gather orientation: coalesced writes, random reads (C4: 481 -> ~130 us vs the
    // scattered-store orientation k_to_user)
    k_from_internal_ilp<<<grid_for((p->n_n + PERM_ILP - 1) / PERM_ILP, 256, 148 * 8), 256, 0,
                          s>>>(p->n_n, p->new_of_old, v_int, v_user);
    LAUNCHED();
}

#ifndef EBS_OUT_PERM
#define EBS_OUT_PERM 0  // 1: SELL writes internal order, then a gather pass to caller order
#endif

// one SELL pass; old_of_new != nullptr: output in caller numbering.  prefilled: `out` was
// already set to -0.0 (fused into to_internal) for the red-mode caller-order output.
void sell_apply(const Plan *p, int mode, const double *x_int, const uint8_t *free_int,
                const int32_t *old_of_new, double *out, cudaStream_t s, bool prefilled = false) {
    double *dst = out;
    const int32_t *o2n = old_of_new;
    const Perm2 *P = nullptr;
    int red = 0;
    if (EBS_PERM2 && old_of_new && p->n_n) {
        // internal-order (coalesced) output, then the two-pass permutation to caller order
        Plan *pm = const_cast<Plan *>(p);
        if ((P = perm_get(pm, 1, s))) {
            dst = plan_vec(pm, OUT_VEC);
            o2n = nullptr;
        }
    }
    if (!P && EBS_OUT_PERM && old_of_new) {
        dst = plan_vec(const_cast<Plan *>(p), 7);
        o2n = nullptr;
    }
    if (o2n && EBS_OUT_RED) {  // red.add into -0.0 (bit-exact, see OpEpi)
        if (!prefilled) fill_negzero(p->n_n, out, s);
        red = 1;
    }
    if (mode == 0) launch_sell_op<0>(p, x_int, free_int, o2n, dst, s, nullptr, nullptr, -1, red);
    else if (mode == 1) launch_sell_op<1>(p, x_int, free_int, o2n, dst, s, nullptr, nullptr, -1, red);
    else launch_sell_op<2>(p, x_int, free_int, o2n, dst, s, nullptr, nullptr, -1, red);
    if (P) {
        perm_apply(const_cast<Plan *>(p), P, dst, out, nullptr, s);
    } else if (EBS_OUT_PERM && old_of_new && p->n_n) {
        k_from_internal_ilp<<<grid_for((p->n_n + PERM_ILP - 1) / PERM_ILP, 256, 148 * 8), 256, 0,
                              s>>>(p->n_n, p->new_of_old, dst, out);
        LAUNCHED();
    }
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_residual(ebs_plan_t plan, const double *x, double *r, int mode, int masked,
                 int32_t *nonfinite, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x && r, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    EBS_REQUIRE(p->has_A && p->has_be, "residual needs an operator loaded with b_e");
    EBS_REQUIRE(mode == EBS_RES_EXACT || mode == EBS_RES_FAST, "bad residual mode %d", mode);
    EBS_REQUIRE(x != r, "x and r must not alias");
    cudaStream_t s = S(stream);
    double *x_int = plan_vec(p, 0);
    if (nonfinite) CU(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), s));
    if (EBS_OUT_RED && EBS_FILL_MODE == 2) fill_negzero(p->n_n, r, s);
    to_internal(p, x, x_int, nonfinite, s, EBS_OUT_RED && EBS_FILL_MODE == 0 ? r : nullptr);
    sell_apply(p, mode == EBS_RES_EXACT ? 2 : 1, x_int, masked ? p->free_int : nullptr,
               p->old_of_new, r, s, EBS_OUT_RED && EBS_FILL_MODE != 1);
    EBS_CATCH
}

int ebs_matvec(ebs_plan_t plan, const double *x, double *y, int masked, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x && y, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(x != y, "x and y must not alias");
    cudaStream_t s = S(stream);
    double *x_int = plan_vec(p, 0);
    if (EBS_OUT_RED && EBS_FILL_MODE == 2) fill_negzero(p->n_n, y, s);
    to_internal(p, x, x_int, nullptr, s, EBS_OUT_RED && EBS_FILL_MODE == 0 ? y : nullptr);
    sell_apply(p, 0, x_int, masked ? p->free_int : nullptr, p->old_of_new, y, s,
               EBS_OUT_RED && EBS_FILL_MODE != 1);
    EBS_CATCH
}

int ebs_to_internal(ebs_plan_t plan, const double *x, double *x_int, int32_t *nonfinite,
                    void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x && x_int, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    if (nonfinite) CU(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), S(stream)));
    to_internal(p, x, x_int, nonfinite, S(stream));
    EBS_CATCH
}

int ebs_to_user(ebs_plan_t plan, const double *v_int, double *v, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && v_int && v, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    to_user(p, v_int, v, S(stream));
    EBS_CATCH
}

int ebs_plan_apply(ebs_plan_t plan, int op, const double *x_int, double *out, int out_user,
                   int masked, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x_int && out, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    EBS_REQUIRE(op >= 0 && op <= 2, "bad op %d", op);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(op == 0 || p->has_be, "residual needs an operator loaded with b_e");
    EBS_REQUIRE(x_int != out, "x and out must not alias");
    EBS_REQUIRE(out_user >= 0 && out_user <= 2, "bad out_user %d", out_user);
    sell_apply(p, op, x_int, masked ? p->free_int : nullptr, out_user ? p->old_of_new : nullptr,
               out, S(stream), out_user == 2);
    EBS_CATCH
}

int ebs_plan_apply_map(ebs_plan_t plan, int op, const double *x_int, double *out,
                       const int32_t *out_map, double *s_raw, int masked, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x_int && out && out_map, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(op == 0 || op == 1, "bad op %d (matvec or fast residual)", op);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(op == 0 || p->has_be, "residual needs an operator loaded with b_e");
    const uint8_t *fm = masked ? p->free_int : nullptr;
    if (op == 0) launch_sell_op<0>(p, x_int, fm, out_map, out, S(stream), s_raw);
    else launch_sell_op<1>(p, x_int, fm, out_map, out, S(stream), s_raw);
    EBS_CATCH
}

int ebs_plan_apply_map_chunks(ebs_plan_t plan, int op, const int32_t *chunks, int64_t n_list,
                              const double *x_int, double *out, const int32_t *out_map,
                              double *s_raw, int masked, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x_int && out && out_map, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(op == 0 || op == 1, "bad op %d (matvec or fast residual)", op);
    EBS_REQUIRE(n_list >= 0 && (chunks || n_list == 0), "bad chunk list");
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(op == 0 || p->has_be, "residual needs an operator loaded with b_e");
    const uint8_t *fm = masked ? p->free_int : nullptr;
    if (op == 0) launch_sell_op<0>(p, x_int, fm, out_map, out, S(stream), s_raw, chunks, n_list);
    else launch_sell_op<1>(p, x_int, fm, out_map, out, S(stream), s_raw, chunks, n_list);
    EBS_CATCH
}

}  // extern "C"

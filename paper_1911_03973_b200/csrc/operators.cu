// operators.cu -- residual / matvec entry points (caller numbering in and out).
//
//   ebs_residual  <- operators.py:72-111 residual (+ operators.py:114-118 mask)
//   ebs_matvec    <- spectrum.py:54-61 _apply_masked
//
// Each call: a gather of x into the plan's internal numbering (with the finiteness check
// of operators.py:90 fused in), a -0.0 fill of the output, then the SELL kernel, whose
// epilogue adds each node's value straight into the caller's numbering.
#include <cstdlib>

#include "sell.cuh"

namespace ebs {

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
            EBS_DCHECK(old_of_new[m] >= 0);
            if (red) atomicAdd(out + old_of_new[m], s);
            else out[old_of_new[m]] = s;
        } else {
            out[m] = s;
        }
    }
};

// Programmatic dependent launch: the SELL pass is launched with programmatic stream
// serialisation, so its CTAs are scheduled while the kernel before it (the -0.0 fill,
// which triggers at its start) drains; griddepcontrol.wait then blocks until that grid
// has completed and its writes are visible.  Without the attribute the wait is a no-op.
// EBS_PDL=0 in the environment launches it the plain way (A/B in profiles/README.md).
template <int NB, int IDS, int MODE>
__global__ void EBS_SELL_BOUNDS(NB)
    k_sell_op(SellView v, const double *__restrict__ x, OpEpi epi) {
    pdl_wait();
    sell_sweep<NB, IDS, MODE == 2>(v, x, epi);
}

template <int NB, int IDS, int MODE>
void launch_sell_op_t(const Plan *p, const double *x_int, const OpEpi &epi, cudaStream_t s,
                      const int32_t *chunks = nullptr, int64_t n_list = -1) {
    auto kern = k_sell_op<NB, IDS, MODE>;
    const SellView v = sell_view(p, chunks, n_list);
    const SellLaunch SL = sell_launch((const void *)kern, NB, p->rowb, v.nlist);
    if (pdl_enabled()) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(SL.grid);
        cfg.blockDim = dim3(SL.block);
        cfg.dynamicSmemBytes = SL.smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, v, x_int, epi);
    } else {
        kern<<<SL.grid, SL.block, SL.smem, s>>>(v, x_int, epi);
    }
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

// caller -> internal numbering: x_int[m] = x_user[old_of_new[m]], 8 independent
// index -> value chains per thread.  The random 8 B reads are L1tex-wavefront bound (~2
// cycles per distinct line; C2 33 us): measured equal or slower were a plain gather, the
// scatter orientation (also with red.add), L2::256B / bulk-L2-prefetch hints and the
// two-pass shared-memory schedule of perm.cu (profiles/README.md).
constexpr int PERM_ILP = 8;

// nonfinite (nullable) is WRITTEN, 0 or 1, by the last block to finish (a block counter and
// an accumulator in the plan's nf_state, both reset by that block): no memset of the flag
// before the launch -- one graph node less per residual.
__global__ void __launch_bounds__(256)
    k_to_internal_ilp(int64_t n, const int32_t *__restrict__ old_of_new,
                      const double *__restrict__ x_user, double *__restrict__ x_int,
                      int32_t *nonfinite, int32_t *state) {
    bool bad = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
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
            EBS_DCHECK(m >= n || (idx[u] >= 0 && idx[u] < n));
            v[u] = m < n ? __ldg(x_user + idx[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PERM_ILP; ++u) {
            const int64_t m = base + u * stride;
            if (m < n) {
                bad |= !isfinite(v[u]);
                x_int[m] = v[u];
            }
        }
    }
    const int any = __syncthreads_or(bad);
    if (nonfinite && threadIdx.x == 0) {
        if (any) atomicOr(state, 1);
        __threadfence();
        const unsigned prev = atomicAdd(reinterpret_cast<unsigned *>(state + 1), 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            *nonfinite = atomicExch(state, 0) ? 1 : 0;
            state[1] = 0;
        }
    }
}

#ifndef EBS_PERM2
// caller <-> internal permutations: 0 direct (random 8 B gather / red-mode scatter),
// 1 the two-pass shared-memory schedule of perm.cu (every global access coalesced),
// 2 automatic: two-pass once a vector outgrows L2's reach.  Fast residual, caller order
// (scripts/perm_crossover.py): direct 177 / 415 / 1166 us vs two-pass 215 / 418 / 827 us
// at 4.2M / 8.4M / 16.8M nodes -- random accesses to DRAM-resident vectors pay 32 B
// sectors for 8 B, the coalesced passes do not.
#define EBS_PERM2 2
#endif
#ifndef EBS_PERM2_MIN_NODES
#define EBS_PERM2_MIN_NODES (8ll << 20)  // 64 MB per vector: the measured crossover
#endif

// the crossover can be overridden by the environment (EBS_PERM2_MIN_NODES, read once):
// tests force either path on small meshes
static int64_t perm2_min_nodes() {
    static const int64_t v = [] {
        const char *e = getenv("EBS_PERM2_MIN_NODES");
        return e ? (int64_t)atoll(e) : (int64_t)EBS_PERM2_MIN_NODES;
    }();
    return v;
}

static bool use_perm2(const Plan *p) {
    if (p->identity) return false;  // identity maps: the direct gather is a coalesced copy
    return EBS_PERM2 == 1 || (EBS_PERM2 == 2 && p->n_n >= perm2_min_nodes());
}

// out[0..n) = value with 16 B stores (scalar head / tail for an unaligned or odd range).
// The -0.0 pre-fill of a red-mode output runs as its own kernel after the x permutation:
// fusing the stores into the latency-bound gather, or running it first, measured slower.
__global__ void k_fill(int64_t n, double value, double *__restrict__ out) {
    pdl_trigger();  // a PDL-launched SELL pass may be scheduled now (it still waits)
    const int64_t head = (reinterpret_cast<uintptr_t>(out) & 15) ? 1 : 0;
    const int64_t n2 = n > head ? (n - head) / 2 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (head && n > 0) out[0] = value;
        if (n > head && ((n - head) & 1)) out[n - 1] = value;
    }
    double2 *o2 = reinterpret_cast<double2 *>(out + head);
    const double2 v = make_double2(value, value);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
         i += (int64_t)gridDim.x * blockDim.x)
        o2[i] = v;
}

static void fill_value(int64_t n, double value, double *out, cudaStream_t s) {
    if (n == 0) return;
    k_fill<<<grid_for((n + 1) / 2, 256, sm_count() * 8), 256, 0, s>>>(n, value, out);
    LAUNCHED();
}

static void fill_negzero(int64_t n, double *out, cudaStream_t s) { fill_value(n, -0.0, out, s); }

void to_internal(const Plan *p, const double *x_user, double *x_int, int32_t *nonfinite,
                 cudaStream_t s, int32_t *nf) {
    if (p->n_n == 0) {
        if (nonfinite) CU(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), s));
        return;
    }
    if (use_perm2(p)) {
        Plan *pm = const_cast<Plan *>(p);
        if (const Perm2 *P = perm_get(pm, 0, s)) {
            if (nonfinite) CU(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), s));
            perm_apply(pm, P, x_user, x_int, nonfinite, s);
            return;
        }
    }
    k_to_internal_ilp<<<grid_for((p->n_n + PERM_ILP - 1) / PERM_ILP, 256, sm_count() * 8), 256, 0, s>>>(
        p->n_n, p->old_of_new, x_user, x_int, nonfinite, nf ? nf : p->nf_state);
    LAUNCHED();
}

// internal -> caller numbering: v_user[i] = v_int[new_of_old[i]] -- coalesced writes,
// random reads (C4: 205 us vs 481 us for the scattered-store orientation)
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
            EBS_DCHECK(i >= n || (idx[u] >= 0 && idx[u] < n));
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
    if (use_perm2(p)) {
        Plan *pm = const_cast<Plan *>(p);
        if (const Perm2 *P = perm_get(pm, 1, s)) {
            perm_apply(pm, P, v_int, v_user, nullptr, s);
            return;
        }
    }
    k_from_internal_ilp<<<grid_for((p->n_n + PERM_ILP - 1) / PERM_ILP, 256, sm_count() * 8), 256, 0,
                          s>>>(p->n_n, p->new_of_old, v_int, v_user);
    LAUNCHED();
}

// one SELL pass; old_of_new != nullptr: output in the caller's numbering (red.add into
// -0.0, filled here unless the caller did: out_user = 2 of ebs_plan_apply)
void sell_apply(const Plan *p, int mode, const double *x_int, const uint8_t *free_int,
                const int32_t *old_of_new, double *out, cudaStream_t s, bool prefilled = false) {
    double *dst = out;
    const int32_t *o2n = p->identity ? nullptr : old_of_new;  // caller order = internal order
    const Perm2 *P = nullptr;
    int red = 0;
    if (use_perm2(p) && o2n && p->n_n) {
        // internal-order (coalesced) output, then the two-pass permutation to caller order
        Plan *pm = const_cast<Plan *>(p);
        if ((P = perm_get(pm, 1, s))) {
            dst = plan_vec(pm, OUT_VEC);
            o2n = nullptr;
        }
    }
    if (o2n && EBS_OUT_RED) {  // red.add into -0.0 (bit-exact, see OpEpi)
        if (!prefilled) fill_negzero(p->n_n, out, s);
        red = 1;
    }
    if (mode == 0) launch_sell_op<0>(p, x_int, free_int, o2n, dst, s, nullptr, nullptr, -1, red);
    else if (mode == 1) launch_sell_op<1>(p, x_int, free_int, o2n, dst, s, nullptr, nullptr, -1, red);
    else launch_sell_op<2>(p, x_int, free_int, o2n, dst, s, nullptr, nullptr, -1, red);
    if (P) perm_apply(const_cast<Plan *>(p), P, dst, out, nullptr, s);
}

// residuals in flight in ebs_residual_many (EBS_MANY_LANES, 1..MANY_MAX; read once)
static int many_lanes() {
    static const int v = [] {
        const char *e = getenv("EBS_MANY_LANES");
        const int l = e ? atoi(e) : 2;
        return l < 1 ? 1 : (l > MANY_MAX ? MANY_MAX : l);
    }();
    return v;
}

void many_free(Plan *p) {
    for (auto &st : p->many_stream) {
        if (st) cudaStreamDestroy(st);
        st = nullptr;
    }
    for (auto &e : p->many_ev) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
    }
}

}  // namespace ebs

using namespace ebs;

extern "C" {

// k independent residuals of device-resident vectors, two in flight: residual i runs on
// the caller's stream (i even) or on the plan's second stream (i odd), each with its own
// internal-order x workspace and non-finite state.  The x permutation and the -0.0 fill of
// one residual (latency-bound, little DRAM traffic) then run while the other's SELL pass
// drains, and the two persistent sweeps fill each other's tails: C2 174 -> 157 us per
// residual (profiles/r02s4_two_stream_probe.log).  Every r_i is the same launch sequence
// as ebs_residual on x_i, so it is bit-identical to it.
int ebs_residual_many(ebs_plan_t plan, const double *x, int64_t ldx, double *r, int64_t ldr,
                      int64_t k, int mode, int masked, int32_t *nonfinite, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && (k == 0 || (x && r)), "null argument");
    EBS_REQUIRE(k >= 0, "negative k");
    Plan *p = reinterpret_cast<Plan *>(plan);
    cudaStream_t s = S(stream);
    OrderGuard order(p->order, s);
    EBS_REQUIRE(p->has_A && p->has_be, "residual needs an operator loaded with b_e");
    EBS_REQUIRE(mode == EBS_RES_EXACT || mode == EBS_RES_FAST, "bad residual mode %d", mode);
    EBS_REQUIRE(ldr >= p->n_n && (ldx == 0 || ldx >= p->n_n),
                "bad leading dimensions (ldx 0 or >= n_nodes, ldr >= n_nodes)");
    EBS_REQUIRE(x != r, "x and r must not alias");
    if (k == 0) return EBS_OK;
    const uint8_t *free_int = masked ? p->free_int : nullptr;
    const int sell_mode = mode == EBS_RES_EXACT ? 2 : 1;
    // the two-pass permutation (meshes beyond L2's reach) stages through plan-held
    // buffers: one residual at a time there
    const int lanes = (k >= 2 && !use_perm2(p)) ? (int)(k < many_lanes() ? k : many_lanes()) : 1;
    if (lanes > 1) {
        if (!p->many_stream[0]) {
            for (auto &st : p->many_stream) CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            for (auto &e : p->many_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        CU(cudaEventRecord(p->many_ev[0], s));  // fork: after the work queued on s
        for (int l = 1; l < lanes; ++l) CU(cudaStreamWaitEvent(p->many_stream[l - 1], p->many_ev[0], 0));
    }
    for (int64_t i = 0; i < k; ++i) {
        const int lane = (int)(i % lanes);
        cudaStream_t st = lane ? p->many_stream[lane - 1] : s;
        double *x_int = plan_vec(p, lane);
        to_internal(p, x + i * ldx, x_int, nonfinite ? nonfinite + i : nullptr, st,
                    p->nf_state + 2 * lane);
        sell_apply(p, sell_mode, x_int, free_int, p->old_of_new, r + i * ldr, st);
    }
    for (int l = 1; l < lanes; ++l) {  // join
        CU(cudaEventRecord(p->many_ev[l], p->many_stream[l - 1]));
        CU(cudaStreamWaitEvent(s, p->many_ev[l], 0));
    }
    EBS_CATCH
}

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
    to_internal(p, x, x_int, nonfinite, s);  // writes *nonfinite (0 / 1)
    sell_apply(p, mode == EBS_RES_EXACT ? 2 : 1, x_int, masked ? p->free_int : nullptr,
               p->old_of_new, r, s);
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
    to_internal(p, x, x_int, nullptr, s);
    sell_apply(p, 0, x_int, masked ? p->free_int : nullptr, p->old_of_new, y, s);
    EBS_CATCH
}

int ebs_to_internal(ebs_plan_t plan, const double *x, double *x_int, int32_t *nonfinite,
                    void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x && x_int, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    OrderGuard order(p->order, S(stream));
    to_internal(p, x, x_int, nonfinite, S(stream));  // writes *nonfinite (0 / 1)
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

int ebs_fill(int64_t n, double value, double *out, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && (out || n == 0), "bad arguments");
    fill_value(n, value, out, S(stream));
    EBS_CATCH
}

int ebs_plan_apply_map_chunks(ebs_plan_t plan, int op, const int32_t *chunks, int64_t n_list,
                              const double *x_int, double *out, const int32_t *out_map,
                              double *s_raw, int flags, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && x_int && out && out_map, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(op == 0 || op == 1, "bad op %d (matvec or fast residual)", op);
    EBS_REQUIRE(n_list >= 0 && (chunks || n_list == 0), "bad chunk list");
    EBS_REQUIRE(flags >= 0 && flags <= 3, "bad flags %d", flags);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    EBS_REQUIRE(op == 0 || p->has_be, "residual needs an operator loaded with b_e");
    const uint8_t *fm = (flags & EBS_APPLY_MASKED) ? p->free_int : nullptr;
    const int red = (flags & EBS_APPLY_ADD) ? 1 : 0;
    if (op == 0)
        launch_sell_op<0>(p, x_int, fm, out_map, out, S(stream), s_raw, chunks, n_list, red);
    else
        launch_sell_op<1>(p, x_int, fm, out_map, out, S(stream), s_raw, chunks, n_list, red);
    EBS_CATCH
}

}  // extern "C"

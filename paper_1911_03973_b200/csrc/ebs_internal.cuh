// ebs_internal.cuh -- shared device/host helpers of libebs.so (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <type_traits>
#include <utility>
#include <stdint.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/ebs.h"

// Device-side index checks (compute-sanitizer is not available on the GPU pool): build
// with -DEBS_DEVICE_CHECKS (scripts/checked_build.sh) and every gather / scatter index of
// the SELL sweeps, permutations, CSR fill and refinement is asserted in range; a violation
// traps the kernel with the file, line and condition.  Compiled out otherwise.
#ifdef EBS_DEVICE_CHECKS
#include <cassert>
#define EBS_DCHECK(cond) assert(cond)
#else
#define EBS_DCHECK(cond) ((void)0)
#endif

namespace ebs {

// ---------------------------------------------------------------- errors ----
void set_error(const char *fmt, ...);
int64_t bump_launches(int64_t n);

struct Fail {
    int code;
};

#define EBS_TRY try {
#define EBS_CATCH                                                                 \
    }                                                                             \
    catch (const ebs::Fail &f) {                                                  \
        return f.code;                                                            \
    }                                                                             \
    catch (...) {                                                                 \
        ebs::set_error("unexpected C++ exception");                               \
        return EBS_ECUDA;                                                         \
    }                                                                             \
    return EBS_OK;

#define EBS_REQUIRE(cond, ...)                                                    \
    do {                                                                          \
        if (!(cond)) {                                                            \
            ebs::set_error(__VA_ARGS__);                                          \
            throw ebs::Fail{EBS_EINVAL};                                          \
        }                                                                         \
    } while (0)

#define CU(call)                                                                  \
    do {                                                                          \
        cudaError_t err_ = (call);                                                \
        if (err_ != cudaSuccess) {                                                \
            cudaGetLastError(); /* a non-sticky error must not resurface later */ \
            ebs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                           cudaGetErrorString(err_));                             \
            throw ebs::Fail{err_ == cudaErrorMemoryAllocation ? EBS_ENOMEM       \
                                                               : EBS_ECUDA};      \
        }                                                                         \
    } while (0)

// launch check: counts one launch of our own kernels
#define LAUNCHED()                                                                \
    do {                                                                          \
        CU(cudaGetLastError());                                                   \
        ebs::bump_launches(1);                                                    \
    } while (0)

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

template <class T>
T *dmalloc(size_t count) {
    T *p = nullptr;
    if (count == 0) count = 1;
    CU(cudaMalloc(&p, count * sizeof(T)));
    return p;
}
template <class T>
void dfree(T *&p) {
    if (p) cudaFree(p);
    p = nullptr;
}

// grid for a 1-D elementwise launch: enough CTAs to fill the 148 SMs several
// times over, grid-stride beyond that
// streaming multiprocessors of the current device (cached per device; 148 on B200)
int sm_count();

inline int grid_for(int64_t n, int block, int max_blocks = -1) {
    if (max_blocks < 0) max_blocks = sm_count() * 16;
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

// ----------------------------------------------------- SELL-32 plan layout ----
constexpr int LANES = 32;                 // nodes per chunk (one warp)
constexpr int J_SHIFT = 30;               // local vertex j packed in the top 2 bits
constexpr int32_t ID_MASK = (1 << J_SHIFT) - 1;

// device-side control block of the solver loop (solve.cu)
struct Ctl {
    int k;              // iteration whose residual was recorded last
    int done;           // 1: later launches are no-ops
    int diverged;
    int n_norms;
    int final_buf;      // ping-pong buffer that holds the returned iterate
    int nonfinite;      // set by any thread writing a non-finite iterate
    int cb_ok;          // r_k of the last step was recorded normally (callback due)
    int x0_nonfinite;   // the solver's x0 held a non-finite entry (reference: ValueError)
    unsigned int counter;  // last-block-done counter of the fused reductions
    unsigned int pad2_;
    double norm0;
    double rz, pq, alpha, beta;
};

// Cross-stream ordering of a shared device workspace.  Calls that use a plan's (or the
// process's) scratch vectors hold the mutex while enqueuing; a call on a different stream
// than the previous one first waits for that call's work (event), so concurrent callers
// on separate streams / host threads are serialised on the device in call order --
// `residual` is safe to call concurrently on a shared batch (reference SPEC.md:273).
// Not applied while the stream is being captured into a CUDA graph (the capture orders).
struct StreamOrder {
    std::recursive_mutex mu;  // recursive: a solver callback may call back into the plan
    cudaEvent_t ev = nullptr;
    cudaStream_t last = nullptr;
    bool rec = false;
};
class OrderGuard {
  public:
    OrderGuard(StreamOrder &o, cudaStream_t s);
    ~OrderGuard();
    OrderGuard(const OrderGuard &) = delete;
    OrderGuard &operator=(const OrderGuard &) = delete;

  private:
    StreamOrder &o_;
    cudaStream_t s_;
    bool active_ = false;
    std::unique_lock<std::recursive_mutex> lk_;
};

// two-pass permutation schedule (perm.cu)
struct Perm2 {
    int64_t n = 0;
    int T = 0;                 // nodes per tile
    uint16_t *src1 = nullptr;  // pass 1: offset in the source tile of the q-th value written
    int32_t *dst1 = nullptr;   // pass 1: its slot in the intermediate (destination-tile order)
    uint16_t *dst2 = nullptr;  // pass 2: offset of intermediate slot k in its destination tile
};

constexpr int MANY_MAX = 4;  // residuals in flight in ebs_residual_many (workspace vectors 0..3)
constexpr int PERM_VEC = 8;  // workspace vector: the permutation intermediate
constexpr int OUT_VEC = 9;   // workspace vector: internal-order operator output

struct Plan {
    int nb;
    int64_t n_n, n_e;
    int64_t n_chunks, n_rows;
    int max_valence;
    // structure
    int32_t *new_of_old = nullptr;  // caller id -> internal id
    int32_t *old_of_new = nullptr;  // internal id -> caller id
    int32_t *cnt = nullptr;         // valence per internal node
    uint8_t *cnt8 = nullptr;        // the same in one byte (max valence <= 255; sweeps read it)
    int32_t *rowbase = nullptr;     // first slot row of each chunk
    int32_t *width = nullptr;       // slot rows of each chunk
    int32_t *slot_ej = nullptr;     // [row][lane]: e | j<<30, -1 for padding
    // slot blob: per row NB planes of 32 doubles (A rows) + the id plane (sell.cuh)
    uint8_t *slot = nullptr;
    int rowb = 0;                   // bytes per slot row
    int packed = 0;                 // id layout: 0 absolute, 1 packed deltas, 2 per-chunk table,
                                    // 3 two-base rows, 4 grid strides
    int32_t *tab = nullptr;         // per-chunk delta tables (layout 2)
    int32_t *taboff = nullptr;      // n_chunks + 1
    // loaded operator
    double *slot_be = nullptr;  // [row][lane]: b_e[j, e] (exact residual)
    double *b_int = nullptr;    // pre-assembled b, internal numbering
    int has_A = 0, has_be = 0;
    // Dirichlet set
    uint8_t *free_int = nullptr;  // 1 free, 0 constrained (internal numbering)
    int64_t n_dirichlet = 0;
    // workspace (lazily grown)
    double *wvec[10] = {nullptr};
    Perm2 perm[2];  // 0: caller -> internal, 1: internal -> caller (built on first use)
    StreamOrder order;  // cross-stream ordering of the workspace above
    // element-slab collectives (nccl.cu): one NCCL communicator per plan
    void *nccl_comm = nullptr;
    int dist_rank = 0, dist_size = 1;
    bool dist_aborted = false;           // ncclCommAbort after an async error / timeout
    const int32_t *dist_stop = nullptr;  // device stop flag of a single-reduction PCG
                                         // (ebs_dist_set_stop): fused matvec sweeps no-op
    double *partials = nullptr;  // reduction partials
    Ctl *ctl = nullptr;          // device control block
    Ctl *ctl_host = nullptr;     // pinned mirror: [0] synchronous reads, [1..2] batch ring
    cudaStream_t cap_stream = nullptr;   // CUDA-graph capture of solver batches (solve.cu)
    cudaEvent_t ring_ev[2] = {nullptr, nullptr};
    double *hist_dev = nullptr;  // device history (norms, errors)
    int64_t hist_cap = 0;
    int32_t *flag = nullptr;     // device scratch flag
    int32_t *nf_state = nullptr; // [accumulator, block counter] of the self-resetting
                                 // non-finite check of the x permutation (operators.cu)
    uint8_t *rowflag = nullptr;  // id layout 3 (3D): 1 per two-base row (sell.cuh IDS_DELTA2)
    int64_t two_base_rows = 0;   // id layout 3: rows coded with two bases
    // single-cluster solver launch (solve.cu k_pcg_cluster), decided once per plan:
    // cl_state 0 unknown, 1 fits (cl_G CTAs of cl_cpb chunks, cl_smem bytes), -1 does not
    int cl_state = 0, cl_G = 0, cl_cpb = 0;
    size_t cl_smem = 0;
    // structured caller numbering (plan.cu find_strides): kept as the internal one
    // (identity maps); every (neighbour - node) id difference is a*stride[0] +
    // b*stride[1] (+ c*stride[2]), a, b, c in {-1, 0, 1}
    bool identity = false;
    int32_t stride[3] = {0, 0, 0};
    // id layout 4 (sell.cuh IDS_TUPLE): per slot a byte indexing the (j, differences) table
    uint8_t *codes = nullptr;
    int4 *tup = nullptr;
    int n_tup = 0;
    void *hostpipe = nullptr;    // host-buffer residual pipeline (hostpipe.cu), lazy
    // ebs_residual_many: the second stream of the two-deep residual pipeline and its
    // fork / join events (operators.cu), lazy
    cudaStream_t many_stream[MANY_MAX - 1] = {nullptr};
    cudaEvent_t many_ev[MANY_MAX] = {nullptr};
};

double *plan_vec(Plan *p, int i);  // workspace vector i (n_n doubles)
StreamOrder &red_order();           // ordering of the per-device reduction scratch
// caller <-> internal numbering (operators.cu)
// nf: the self-resetting state of the non-finite check (2 ints; default the plan's first pair)
void to_internal(const Plan *p, const double *x_user, double *x_int, int32_t *nonfinite,
                 cudaStream_t s, int32_t *nf = nullptr);
void many_free(Plan *p);
void to_user(const Plan *p, const double *v_int, double *v_user, cudaStream_t s);
const Perm2 *perm_get(Plan *p, int dir, cudaStream_t s);
void perm_apply(Plan *p, const Perm2 *P, const double *in, double *out, int32_t *nonfinite,
                cudaStream_t s);
void perm_free(Plan *p);
void dist_free(Plan *p);
void hostpipe_free(Plan *p);

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream
// serialisation is scheduled while its predecessor drains; griddepcontrol.wait at its
// entry then blocks until the predecessor grid has completed and its writes are visible
// (a no-op for a plain launch).  EBS_PDL=0 in the environment disables it everywhere.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// launch `kern` on `s`, with programmatic stream serialisation when pdl_enabled()
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CU(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ------------------------------------------------------ reductions ----------
constexpr int RED_BLOCK = 256;
// occupancy-sized grid of `kernel` (one wave of resident CTAs, cached per kernel and
// device; sell.cuh repeats the declaration with smem defaulted to 0)
int persistent_grid(const void *kernel, int block, int64_t work_blocks, size_t smem);
constexpr int RED_MAX_BLOCKS = 1184;  // 148 SMs x 8: fixed -> deterministic order

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum of NV values (fixed tree).  Result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *smem /*[NV*32]*/) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) smem[q * 32 + wid] = v[q];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double t = lane < nw ? smem[q * 32 + lane] : 0.0;
            v[q] = warp_sum(t);
        }
    }
}

// Last-block-done pattern: every block writes its NV partial sums; the last block
// to arrive sums all partials in block order and returns true in ALL its threads
// with the totals in tot[] (valid in thread 0).  Deterministic for a fixed grid.
template <int NV>
__device__ __forceinline__ bool grid_sum_last(double (&v)[NV], double *partials,
                                              unsigned int *counter, double (&tot)[NV]) {
    __shared__ double smem[NV * 32];
    __shared__ bool am_last;
    block_sum<NV>(v, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) partials[(size_t)q * gridDim.x + blockIdx.x] = v[q];
        __threadfence();
        unsigned int prev = atomicAdd(counter, 1u);
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return false;
    __threadfence();
    double w[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
            s += __ldcg(&partials[(size_t)q * gridDim.x + b]);
        w[q] = s;
    }
    block_sum<NV>(w, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) tot[q] = w[q];
        *counter = 0u;  // re-arm for the next launch (stream order)
    }
    return true;
}

}  // namespace ebs

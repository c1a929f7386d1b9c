// hostpipe.cu -- residuals of k caller-numbered vectors that live in HOST memory.
//
//   ebs_residual_many_host <- operators.py:72-111 residual, called k times on host arrays
//
// The reference evaluates `residual(batch, x)` on NumPy arrays; a caller that keeps its
// vectors on the host pays a host->device copy of x and a device->host copy of r per
// call.  At C2 size (33.6 MB each way) those copies take ~0.6 ms apiece on PCIe 5 x16
// against 0.17 ms of residual, so the call is a pipeline: the H2D of x_{i+1}, the
// residual of x_i and the D2H of r_{i-1} run concurrently on three streams (two copy
// engines, one for each direction, and the caller's stream for the kernels), NB device
// buffers per side.  Each r_i is bit-identical to ebs_residual on x_i (the same call
// runs on the device buffers).
#include <cstdlib>

#include "ebs_internal.cuh"

namespace ebs {

constexpr int PIPE_MAX = 4;

struct HostPipe {
    int nb = 0;
    int64_t n = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    double *xb[PIPE_MAX] = {}, *rb[PIPE_MAX] = {};
    cudaEvent_t x_in[PIPE_MAX] = {}, used[PIPE_MAX] = {}, r_read[PIPE_MAX] = {};
    cudaEvent_t start = nullptr, d2h_done = nullptr;
    int32_t *flags = nullptr;
    int64_t flags_cap = 0;
};

// buffers per side (EBS_PIPE_NB, 2..4; 3 by default: profiles/r02_e2e_pipeline.txt)
static int pipe_depth() {
    static int nb = [] {
        const char *e = getenv("EBS_PIPE_NB");
        int v = e ? atoi(e) : 3;
        return v < 2 ? 2 : (v > PIPE_MAX ? PIPE_MAX : v);
    }();
    return nb;
}

void hostpipe_free(Plan *p) {
    auto *hp = reinterpret_cast<HostPipe *>(p->hostpipe);
    if (!hp) return;
    for (int j = 0; j < PIPE_MAX; ++j) {
        dfree(hp->xb[j]);
        dfree(hp->rb[j]);
        for (cudaEvent_t e : {hp->x_in[j], hp->used[j], hp->r_read[j]})
            if (e) cudaEventDestroy(e);
    }
    if (hp->start) cudaEventDestroy(hp->start);
    if (hp->d2h_done) cudaEventDestroy(hp->d2h_done);
    if (hp->h2d) cudaStreamDestroy(hp->h2d);
    if (hp->d2h) cudaStreamDestroy(hp->d2h);
    dfree(hp->flags);
    delete hp;
    p->hostpipe = nullptr;
}

static HostPipe *hostpipe_get(Plan *p, int64_t k) {
    auto *hp = reinterpret_cast<HostPipe *>(p->hostpipe);
    if (!hp) {
        hp = new HostPipe();
        p->hostpipe = hp;
        hp->nb = pipe_depth();
        hp->n = p->n_n;
        CU(cudaStreamCreateWithFlags(&hp->h2d, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&hp->d2h, cudaStreamNonBlocking));
        for (int j = 0; j < hp->nb; ++j) {
            hp->xb[j] = dmalloc<double>(p->n_n);
            hp->rb[j] = dmalloc<double>(p->n_n);
            for (cudaEvent_t *e : {&hp->x_in[j], &hp->used[j], &hp->r_read[j]})
                CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        CU(cudaEventCreateWithFlags(&hp->start, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&hp->d2h_done, cudaEventDisableTiming));
    }
    if (k > hp->flags_cap) {
        dfree(hp->flags);
        hp->flags = dmalloc<int32_t>(k);
        hp->flags_cap = k;
    }
    return hp;
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_residual_many_host(ebs_plan_t plan, const double *x_host, int64_t ldx, double *r_host,
                           int64_t ldr, int64_t k, int mode, int masked, int32_t *nonfinite_host,
                           void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && (k == 0 || (x_host && r_host)), "null argument");
    EBS_REQUIRE(k >= 0, "negative k");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A && p->has_be, "residual needs an operator loaded with b_e");
    EBS_REQUIRE(mode == EBS_RES_EXACT || mode == EBS_RES_FAST, "bad residual mode %d", mode);
    EBS_REQUIRE(ldx >= 0 && ldr >= p->n_n, "bad leading dimensions (ldx >= 0, ldr >= n_nodes)");
    EBS_REQUIRE(k <= 1 || ldx == 0 || ldx >= p->n_n, "ldx must be 0 or >= n_nodes");
    cudaStream_t s = S(stream);
    OrderGuard order(p->order, s);  // the pipeline's buffers are the plan's: one caller at a time
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(s, &st));
    EBS_REQUIRE(st == cudaStreamCaptureStatusNone,
                "ebs_residual_many_host synchronises the host; it cannot be graph-captured");
    if (k == 0) return EBS_OK;
    const size_t bytes = (size_t)p->n_n * sizeof(double);
    HostPipe *hp = hostpipe_get(p, k);
    const int nb = hp->nb;
    // the copy streams start after the work already queued on the caller's stream
    CU(cudaEventRecord(hp->start, s));
    CU(cudaStreamWaitEvent(hp->h2d, hp->start, 0));
    CU(cudaStreamWaitEvent(hp->d2h, hp->start, 0));
    for (int64_t i = 0; i < k; ++i) {
        const int j = (int)(i % nb);
        if (i >= nb) CU(cudaStreamWaitEvent(hp->h2d, hp->used[j], 0));  // x_{i-nb} consumed
        if (bytes) CU(cudaMemcpyAsync(hp->xb[j], x_host + i * ldx, bytes, cudaMemcpyHostToDevice, hp->h2d));
        CU(cudaEventRecord(hp->x_in[j], hp->h2d));
        CU(cudaStreamWaitEvent(s, hp->x_in[j], 0));
        if (i >= nb) CU(cudaStreamWaitEvent(s, hp->r_read[j], 0));  // r_{i-nb} read back
        int rc = ebs_residual(plan, hp->xb[j], hp->rb[j], mode, masked,
                              nonfinite_host ? hp->flags + i : nullptr, stream);
        if (rc != EBS_OK) throw Fail{rc};
        CU(cudaEventRecord(hp->used[j], s));
        CU(cudaStreamWaitEvent(hp->d2h, hp->used[j], 0));
        if (bytes) CU(cudaMemcpyAsync(r_host + i * ldr, hp->rb[j], bytes, cudaMemcpyDeviceToHost, hp->d2h));
        CU(cudaEventRecord(hp->r_read[j], hp->d2h));
    }
    CU(cudaEventRecord(hp->d2h_done, hp->d2h));
    CU(cudaStreamWaitEvent(s, hp->d2h_done, 0));
    if (nonfinite_host)
        CU(cudaMemcpyAsync(nonfinite_host, hp->flags, k * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    EBS_CATCH
}

}  // extern "C"

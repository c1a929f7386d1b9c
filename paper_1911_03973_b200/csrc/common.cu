// common.cu -- error reporting, launch counter and small vector kernels of libebs.so.
#include <atomic>
#include <cstdarg>
#include <mutex>

#include "ebs_internal.cuh"

namespace ebs {

static thread_local char g_err[1024] = {0};
static std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int64_t bump_launches(int64_t n) { return g_launches.fetch_add(n) + n; }

// ------------------------------------------------------------- kernels ------
__global__ void k_dot(int64_t n, const double *__restrict__ x, const double *__restrict__ y,
                      double *partials, unsigned int *counter, double *out, int sqrt_it) {
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[0] += x[i] * y[i];
    double tot[1];
    if (grid_sum_last<1>(v, partials, counter, tot) && threadIdx.x == 0)
        *out = sqrt_it ? sqrt(tot[0]) : tot[0];
}

__global__ void k_axpby(int64_t n, double a, const double *__restrict__ x, double b,
                        double *__restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = a * x[i] + b * y[i];
}

__global__ void k_mask(int64_t n, const double *__restrict__ v, int64_t n_d,
                       const int64_t *__restrict__ nd, double *__restrict__ out, int pass) {
    if (pass == 0) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x)
            out[i] = v[i];
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_d;
             i += (int64_t)gridDim.x * blockDim.x) {
            int64_t k = nd[i];
            if (k >= 0 && k < n) out[k] = 0.0;
        }
    }
}

__global__ void k_check_finite(int64_t n, const double *__restrict__ v, int32_t *flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(v[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void k_gather(int64_t n, const int64_t *__restrict__ idx,
                         const double *__restrict__ v, double *__restrict__ buf) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = v[idx[i]];
}

__global__ void k_scatter_add(int64_t n, const int64_t *__restrict__ idx,
                              const double *__restrict__ buf, double *__restrict__ v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[idx[i]] += buf[i];
}

int sm_count() {
    static int cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    int &c = cache[dev & 63];
    if (c == 0 && cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        c = 148;
    return c;
}

// occupancy-sized persistent grid, cached per (kernel, device)
bool pdl_enabled() {
    static const bool v = [] {
        const char *e = getenv("EBS_PDL");
        return !(e && e[0] == '0');
    }();
    return v;
}

int persistent_grid(const void *kernel, int block, int64_t work_blocks, size_t smem) {
    struct Ent { const void *k; int dev; int block; size_t smem; int grid; };
    static Ent cache[64];
    static int n_cache = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    CU(cudaGetDevice(&dev));
    int grid = -1;
    for (int i = 0; i < n_cache; ++i)
        if (cache[i].k == kernel && cache[i].dev == dev && cache[i].block == block &&
            cache[i].smem == smem)
            grid = cache[i].grid;
    if (grid < 0) {
        int per_sm = 0, sms = 0;
        if (smem > 48 * 1024)
            CU(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        grid = (per_sm > 0 ? per_sm : 1) * sms;
        if (grid > 8192) grid = 8192;
        if (n_cache < 64) cache[n_cache++] = Ent{kernel, dev, block, smem, grid};
    }
    if (work_blocks < 1) work_blocks = 1;
    return (int)(work_blocks < grid ? work_blocks : grid);
}

}  // namespace ebs
#include "sell.cuh"
namespace ebs {

SellLaunch sell_launch(const void *kernel, int nb, int rowb, int64_t n_chunks) {
    SellLaunch L;
#if EBS_TMA
    const int W = nb == 3 ? TmaCfg<3>::W : TmaCfg<4>::W;
    const int R = nb == 3 ? TmaCfg<3>::R : TmaCfg<4>::R;
    const int S = nb == 3 ? TmaCfg<3>::S : TmaCfg<4>::S;
    L.block = W * LANES;
    L.smem = (size_t)W * S * R * rowb;
    L.grid = persistent_grid(kernel, L.block, (n_chunks + W - 1) / W, L.smem);
#else
    (void)rowb;
    L.block = 256;
    L.smem = 0;
    L.grid = persistent_grid(kernel, 256, (n_chunks * LANES + 255) / 256, 0);
#endif
    return L;
}

OrderGuard::OrderGuard(StreamOrder &o, cudaStream_t s) : o_(o), s_(s), lk_(o.mu) {
#ifdef EBS_NO_ORDER  // test builds only: demonstrates the race the guard prevents
    return;
#endif
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    active_ = st == cudaStreamCaptureStatusNone;
    if (!active_) return;
    if (!o_.ev) CU(cudaEventCreateWithFlags(&o_.ev, cudaEventDisableTiming));
    if (o_.rec && o_.last != s) CU(cudaStreamWaitEvent(s, o_.ev, 0));
}

OrderGuard::~OrderGuard() {
    if (!active_) return;
    if (cudaEventRecord(o_.ev, s_) == cudaSuccess) {
        o_.last = s_;
        o_.rec = true;
    } else {
        cudaGetLastError();
    }
}

// scratch for the standalone reductions, one per device; callers hold red_order(dev)
constexpr int MAX_DEV = 64;
static double *g_partials[MAX_DEV] = {};
static unsigned int *g_counter[MAX_DEV] = {};
static StreamOrder g_red_order[MAX_DEV];

StreamOrder &red_order() {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    return g_red_order[dev % MAX_DEV];
}

void reduce_scratch(double **partials, unsigned int **counter) {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    dev %= MAX_DEV;
    if (!g_partials[dev]) {
        CU(cudaMalloc(&g_partials[dev], sizeof(double) * 4 * RED_MAX_BLOCKS));
        CU(cudaMalloc(&g_counter[dev], sizeof(unsigned int) * 4));
        CU(cudaMemset(g_counter[dev], 0, sizeof(unsigned int) * 4));
    }
    *partials = g_partials[dev];
    *counter = g_counter[dev];
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_version(void) { return 100; }

int ebs_last_error(char *buf, size_t len) {
    if (!buf || len == 0) return EBS_EINVAL;
    strncpy(buf, g_err, len - 1);
    buf[len - 1] = 0;
    return EBS_OK;
}

int64_t ebs_launch_count(void) { return g_launches.load(); }

int ebs_dot(int64_t n, const double *x, const double *y, double *out, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && out, "ebs_dot: bad arguments");
    double *partials;
    unsigned int *counter;
    OrderGuard order(red_order(), S(stream));
    reduce_scratch(&partials, &counter);
    k_dot<<<grid_for(n, RED_BLOCK, RED_MAX_BLOCKS), RED_BLOCK, 0, S(stream)>>>(
        n, x, y, partials, counter, out, 0);
    LAUNCHED();
    EBS_CATCH
}

int ebs_nrm2(int64_t n, const double *x, double *out, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && out, "ebs_nrm2: bad arguments");
    double *partials;
    unsigned int *counter;
    OrderGuard order(red_order(), S(stream));
    reduce_scratch(&partials, &counter);
    k_dot<<<grid_for(n, RED_BLOCK, RED_MAX_BLOCKS), RED_BLOCK, 0, S(stream)>>>(
        n, x, x, partials, counter, out, 1);
    LAUNCHED();
    EBS_CATCH
}

int ebs_axpby(int64_t n, double a, const double *x, double b, double *y, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "ebs_axpby: bad n");
    if (n == 0) return EBS_OK;
    k_axpby<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, a, x, b, y);
    LAUNCHED();
    EBS_CATCH
}

int ebs_mask(int64_t n, const double *v, int64_t n_d, const int64_t *nd, double *out,
             void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && n_d >= 0, "ebs_mask: bad sizes");
    if (n > 0 && v != out) {
        k_mask<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, v, n_d, nd, out, 0);
        LAUNCHED();
    }
    if (n_d > 0) {
        k_mask<<<grid_for(n_d, 256), 256, 0, S(stream)>>>(n, v, n_d, nd, out, 1);
        LAUNCHED();
    }
    EBS_CATCH
}

int ebs_check_finite(int64_t n, const double *v, int32_t *flag, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0 && flag, "ebs_check_finite: bad arguments");
    CU(cudaMemsetAsync(flag, 0, sizeof(int32_t), S(stream)));
    if (n > 0) {
        k_check_finite<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, v, flag);
        LAUNCHED();
    }
    EBS_CATCH
}

int ebs_gather(int64_t n, const int64_t *idx, const double *v, double *buf, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "ebs_gather: bad n");
    if (n == 0) return EBS_OK;
    k_gather<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, idx, v, buf);
    LAUNCHED();
    EBS_CATCH
}

int ebs_scatter_add(int64_t n, const int64_t *idx, const double *buf, double *v,
                    void *stream) {
    EBS_TRY
    EBS_REQUIRE(n >= 0, "ebs_scatter_add: bad n");
    if (n == 0) return EBS_OK;
    k_scatter_add<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, idx, buf, v);
    LAUNCHED();
    EBS_CATCH
}

}  // extern "C"

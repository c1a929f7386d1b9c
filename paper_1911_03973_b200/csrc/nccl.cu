// nccl.cu -- the element-slab collectives inside libebs.so (ebs_dist_init and
// the halo exchange), for callers that drive the multi-GPU path from C without Python.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): in a PyTorch process that is the
// library torch already loaded, elsewhere the system one -- libebs.so never links a second
// NCCL into a process.  One communicator per plan (one rank = one GPU = one element slab).
//
//   ebs_dist_unique_id  ncclGetUniqueId (rank 0; the caller broadcasts the 128 bytes)
//   ebs_dist_init       ncclCommInitRank on the current device, stored in the plan
//   ebs_dist_exchange   grouped ncclSend / ncclRecv of per-peer device buffers on `stream`
//                       (the interface partial sums of the slab neighbours)
//   ebs_dist_allreduce  in-place ncclAllReduce(sum) of doubles on `stream`
//   ebs_dist_poll       ncclCommGetAsyncError: a failed peer / network error -> abort
//   ebs_dist_wait       wait for `stream` while polling for async errors, abort on timeout
//   ebs_dist_abort      ncclCommAbort: pending collectives return, the plan's comm is dead
// A lost peer never hangs the caller that waits through ebs_dist_wait: the communicator is
// aborted (ncclCommAbort unblocks the NCCL kernels in flight) and EBS_ENCCL returned.
#include <dlfcn.h>

#include <chrono>
#include <thread>
#include <nccl.h>

#include "ebs_internal.cuh"

namespace ebs {

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
    ncclResult_t (*getAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char *e = dlerror();
            api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        bool all = true;
        auto sym = [&](auto &fn, const char *name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) {
                all = false;
                api.why += std::string(" missing ") + name;
            }
        };
        sym(api.getUniqueId, "ncclGetUniqueId");
        sym(api.commInitRank, "ncclCommInitRank");
        sym(api.commDestroy, "ncclCommDestroy");
        sym(api.groupStart, "ncclGroupStart");
        sym(api.groupEnd, "ncclGroupEnd");
        sym(api.send, "ncclSend");
        sym(api.recv, "ncclRecv");
        sym(api.allReduce, "ncclAllReduce");
        sym(api.errorString, "ncclGetErrorString");
        sym(api.getAsyncError, "ncclCommGetAsyncError");
        sym(api.commAbort, "ncclCommAbort");
        api.ok = all;
    });
    return api;
}

#define NC(call)                                                                   \
    do {                                                                           \
        ncclResult_t r_ = (call);                                                  \
        if (r_ != ncclSuccess) {                                                   \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                   \
                      nccl().errorString ? nccl().errorString(r_) : "nccl error"); \
            throw Fail{EBS_ENCCL};                                                 \
        }                                                                          \
    } while (0)

const NcclApi &need_nccl() {
    const NcclApi &a = nccl();
    if (!a.ok) {
        set_error("NCCL unavailable:%s", a.why.c_str());
        throw Fail{EBS_ENCCL};
    }
    return a;
}

}  // namespace

// the plan's live communicator, or EBS_ENCCL (never initialised / aborted)
ncclComm_t live_comm(Plan *p) {
    if (p->dist_aborted) {
        set_error("the plan's NCCL communicator was aborted (async error or timeout)");
        throw Fail{EBS_ENCCL};
    }
    if (!p->nccl_comm) {
        set_error("ebs_dist_init first");
        throw Fail{EBS_ENCCL};
    }
    return static_cast<ncclComm_t>(p->nccl_comm);
}

void abort_comm(Plan *p) {
    if (p->nccl_comm && !p->dist_aborted && nccl().ok)
        nccl().commAbort(static_cast<ncclComm_t>(p->nccl_comm));
    p->dist_aborted = true;
}

// ncclCommGetAsyncError; on an error the communicator is aborted and EBS_ENCCL thrown
void poll_comm(Plan *p) {
    ncclComm_t comm = live_comm(p);
    const NcclApi &a = need_nccl();
    ncclResult_t st = ncclSuccess;
    ncclResult_t r = a.getAsyncError(comm, &st);
    if (r != ncclSuccess || (st != ncclSuccess && st != ncclInProgress)) {
        const ncclResult_t e = r != ncclSuccess ? r : st;
        abort_comm(p);
        set_error("NCCL asynchronous error: %s (communicator aborted)", a.errorString(e));
        throw Fail{EBS_ENCCL};
    }
}

void dist_free(Plan *p) {
    if (p->nccl_comm && nccl().ok) {
        if (p->dist_aborted) {
            // ncclCommAbort already released it
        } else {
            nccl().commDestroy(static_cast<ncclComm_t>(p->nccl_comm));
        }
    }
    p->nccl_comm = nullptr;
    p->dist_aborted = false;
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_dist_unique_id(void *id_out) {
    EBS_TRY
    EBS_REQUIRE(id_out, "null argument");
    static_assert(sizeof(ncclUniqueId) == EBS_DIST_ID_BYTES, "ncclUniqueId size");
    const NcclApi &a = need_nccl();
    ncclUniqueId id;
    NC(a.getUniqueId(&id));
    memcpy(id_out, &id, sizeof id);
    EBS_CATCH
}

int ebs_dist_init(ebs_plan_t plan, const void *id, int rank, int nranks) {
    EBS_TRY
    EBS_REQUIRE(plan && id, "null argument");
    EBS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d of %d", rank, nranks);
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(!p->nccl_comm || p->dist_aborted, "the plan already has a communicator");
    if (p->dist_aborted) dist_free(p);  // re-initialisation after an abort
    const NcclApi &a = need_nccl();
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    NC(a.commInitRank(&comm, nranks, uid, rank));
    p->nccl_comm = comm;
    p->dist_rank = rank;
    p->dist_size = nranks;
    EBS_CATCH
}

int ebs_dist_exchange(ebs_plan_t plan, int n_peers, const int32_t *peers, const int64_t *counts,
                      const double *const *send, double *const *recv, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && (n_peers == 0 || (peers && counts && send && recv)), "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    ncclComm_t comm = live_comm(p);
    for (int i = 0; i < n_peers; ++i) {
        EBS_REQUIRE(peers[i] >= 0 && peers[i] < p->dist_size, "bad peer %d", peers[i]);
        EBS_REQUIRE(counts[i] >= 0 && (counts[i] == 0 || (send[i] && recv[i])),
                    "bad buffers for peer %d", peers[i]);
    }
    if (n_peers == 0) return EBS_OK;
    const NcclApi &a = need_nccl();
    NC(a.groupStart());
    ncclResult_t first = ncclSuccess;
    for (int i = 0; i < n_peers && first == ncclSuccess; ++i) {
        if (counts[i] == 0) continue;
        first = a.send(send[i], (size_t)counts[i], ncclDouble, peers[i], comm, S(stream));
        if (first == ncclSuccess)
            first = a.recv(recv[i], (size_t)counts[i], ncclDouble, peers[i], comm, S(stream));
    }
    ncclResult_t end = a.groupEnd();
    NC(first);
    NC(end);
    EBS_CATCH
}

int ebs_dist_allreduce(ebs_plan_t plan, double *buf, int64_t n, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && (buf || n == 0) && n >= 0, "bad arguments");
    Plan *p = reinterpret_cast<Plan *>(plan);
    ncclComm_t comm = live_comm(p);
    if (n == 0) return EBS_OK;
    const NcclApi &a = need_nccl();
    NC(a.allReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, comm, S(stream)));
    EBS_CATCH
}

int ebs_dist_poll(ebs_plan_t plan) {
    EBS_TRY
    EBS_REQUIRE(plan, "null argument");
    poll_comm(reinterpret_cast<Plan *>(plan));
    EBS_CATCH
}

int ebs_dist_wait(ebs_plan_t plan, void *stream, double timeout_s) {
    EBS_TRY
    EBS_REQUIRE(plan, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    poll_comm(p);
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; ++spin) {
        cudaError_t q = cudaStreamQuery(S(stream));
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) CU(q);
        poll_comm(p);
        const double el =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_s >= 0.0 && el > timeout_s) {
            abort_comm(p);
            set_error("stream not complete after %.1f s (lost peer?): NCCL communicator "
                      "aborted", el);
            return EBS_ENCCL;
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    poll_comm(p);
    EBS_CATCH
}

int ebs_dist_abort(ebs_plan_t plan) {
    EBS_TRY
    EBS_REQUIRE(plan, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->nccl_comm, "no communicator");
    abort_comm(p);
    EBS_CATCH
}

}  // extern "C"

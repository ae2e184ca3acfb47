// comm.cu -- the path's only collective: the BWW weight-gradient exchange of
// batch-sharded training.
//
// FWD and BWI are independent per image, so a rank runs its contiguous batch
// slice of ActNCHWc with no communication.  BWW sums over images: every rank
// computes the partial dG of its slice and the ranks sum it with one NCCL
// allreduce (fp32, in place) over NVLink / NVSwitch.  The reference has no
// distributed layer (its only concurrency is the per-call worker pool,
// P/src/kernels.cpp:76-102); this is the B200-side addition BASELINE asks for.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a process that
// already loaded PyTorch's NCCL the same library instance is reused (one NCCL
// per process), and the product library still loads where NCCL is absent
// (every comm entry then returns SPC_ERR_NCCL).
//
// Symmetric windows: spc_comm_window_alloc places a buffer in ncclMemAlloc
// memory registered with ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC), so
// the BWW split reduction writes dG straight into memory NCCL's symmetric
// kernels read from its peers over NVLink, and spc_bww_sharded enqueues the
// allreduce right behind the reduction on the same stream (no host sync).
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace spc {
spc_status set_error(spc_status st, const std::string& msg);
}

namespace {

// The subset of nccl.h this file needs (ABI-stable since NCCL 2.0; windows 2.27).
typedef int ncclResult_t;
typedef void* ncclComm_t;
typedef void* ncclWindow_t;
struct ncclUniqueId { char internal[128]; };
enum { ncclSuccess = 0 };
enum { ncclFloat32 = 7, ncclUint64 = 5 };
enum { ncclSum = 0 };
constexpr int NCCL_WIN_COLL_SYMMETRIC = 0x01;

struct NcclApi {
    bool ok = false;
    std::string why;
    int version = 0;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*MemFree)(void*) = nullptr;
    ncclResult_t (*WindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not loadable: ") + (dlerror() ? dlerror() : "?");
            return;
        }
#define SPC_SYM(field, name)                                          \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
    if (!api.field) {                                                  \
        api.why = std::string("NCCL symbol missing: ") + name;         \
        return;                                                        \
    }
        SPC_SYM(GetVersion, "ncclGetVersion");
        SPC_SYM(GetUniqueId, "ncclGetUniqueId");
        SPC_SYM(CommInitRank, "ncclCommInitRank");
        SPC_SYM(CommDestroy, "ncclCommDestroy");
        SPC_SYM(CommCount, "ncclCommCount");
        SPC_SYM(CommUserRank, "ncclCommUserRank");
        SPC_SYM(AllReduce, "ncclAllReduce");
        SPC_SYM(MemAlloc, "ncclMemAlloc");
        SPC_SYM(MemFree, "ncclMemFree");
        SPC_SYM(GetErrorString, "ncclGetErrorString");
#undef SPC_SYM
        // windows are optional (NCCL >= 2.27): without them buffers are plain ncclMemAlloc
        api.WindowRegister = reinterpret_cast<decltype(api.WindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
        api.WindowDeregister =
            reinterpret_cast<decltype(api.WindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
        api.GetVersion(&api.version);
        api.ok = true;
    });
    return api;
}

spc_status nccl_fail(ncclResult_t r, const char* where) {
    NcclApi& a = nccl();
    return spc::set_error(SPC_ERR_NCCL, std::string(where) + ": " +
                                            (a.GetErrorString ? a.GetErrorString(r) : "nccl error"));
}

spc_status need_nccl() {
    NcclApi& a = nccl();
    return a.ok ? SPC_OK : spc::set_error(SPC_ERR_NCCL, a.why);
}

}  // namespace

struct spc_comm {
    ncclComm_t nc = nullptr;
    bool owned = false;
    int nranks = 1, rank = 0, device = 0;
    struct Win {
        void* ptr;
        size_t bytes;
        ncclWindow_t win;
    };
    std::mutex mu;
    std::vector<Win> wins;
};

extern "C" {

int spc_nccl_version(void) {
    NcclApi& a = nccl();
    return a.ok ? a.version : 0;
}

spc_status spc_comm_unique_id(unsigned char* id_out) {
    if (!id_out) return spc::set_error(SPC_ERR_ARG, "null id buffer");
    if (spc_status s = need_nccl()) return s;
    ncclUniqueId id;
    if (ncclResult_t r = nccl().GetUniqueId(&id)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, SPC_COMM_ID_BYTES);
    return SPC_OK;
}

spc_status spc_comm_init(spc_comm** out, int nranks, const unsigned char* id, int rank) {
    if (!out || !id) return spc::set_error(SPC_ERR_ARG, "null comm or id");
    if (nranks < 1 || rank < 0 || rank >= nranks) return spc::set_error(SPC_ERR_ARG, "bad nranks/rank");
    if (spc_status s = need_nccl()) return s;
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, SPC_COMM_ID_BYTES);
    spc_comm* c = new spc_comm;
    cudaGetDevice(&c->device);
    if (ncclResult_t r = nccl().CommInitRank(&c->nc, nranks, uid, rank)) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    c->owned = true;
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return SPC_OK;
}

spc_status spc_comm_wrap(spc_comm** out, void* nccl_comm) {
    if (!out || !nccl_comm) return spc::set_error(SPC_ERR_ARG, "null comm");
    if (spc_status s = need_nccl()) return s;
    spc_comm* c = new spc_comm;
    c->nc = nccl_comm;
    cudaGetDevice(&c->device);
    nccl().CommCount(c->nc, &c->nranks);
    nccl().CommUserRank(c->nc, &c->rank);
    *out = c;
    return SPC_OK;
}

void* spc_comm_nccl(spc_comm* comm) { return comm ? comm->nc : nullptr; }
int spc_comm_size(spc_comm* comm) { return comm ? comm->nranks : 0; }
int spc_comm_rank(spc_comm* comm) { return comm ? comm->rank : -1; }

spc_status spc_comm_destroy(spc_comm* comm) {
    if (!comm) return SPC_OK;
    spc_status st = SPC_OK;
    for (auto& w : comm->wins) {
        if (w.win && nccl().WindowDeregister) nccl().WindowDeregister(comm->nc, w.win);
        nccl().MemFree(w.ptr);
    }
    if (comm->owned) {
        if (ncclResult_t r = nccl().CommDestroy(comm->nc)) st = nccl_fail(r, "ncclCommDestroy");
    }
    delete comm;
    return st;
}

// Collective: every rank calls it with the same size, in the same order.
spc_status spc_comm_window_alloc(spc_comm* comm, size_t bytes, void** ptr, int* symmetric) {
    if (!comm || !ptr) return spc::set_error(SPC_ERR_ARG, "null comm or ptr");
    if (spc_status s = need_nccl()) return s;
    void* p = nullptr;
    if (ncclResult_t r = nccl().MemAlloc(&p, bytes ? bytes : 4)) return nccl_fail(r, "ncclMemAlloc");
    ncclWindow_t win = nullptr;
    int sym = 0;
    // The window is an optimisation (NCCL's symmetric kernels); where the
    // library or the system cannot register one, the buffer stays plain
    // ncclMemAlloc memory and the allreduce takes NCCL's regular path.
    if (nccl().WindowRegister &&
        nccl().WindowRegister(comm->nc, p, bytes ? bytes : 4, &win, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess)
        sym = 1;
    else
        win = nullptr;
    {
        std::lock_guard<std::mutex> g(comm->mu);
        comm->wins.push_back({p, bytes, win});
    }
    *ptr = p;
    if (symmetric) *symmetric = sym;
    return SPC_OK;
}

spc_status spc_comm_window_free(spc_comm* comm, void* ptr) {
    if (!comm || !ptr) return spc::set_error(SPC_ERR_ARG, "null comm or ptr");
    std::lock_guard<std::mutex> g(comm->mu);
    for (size_t i = 0; i < comm->wins.size(); ++i) {
        if (comm->wins[i].ptr != ptr) continue;
        if (comm->wins[i].win && nccl().WindowDeregister) nccl().WindowDeregister(comm->nc, comm->wins[i].win);
        nccl().MemFree(ptr);
        comm->wins.erase(comm->wins.begin() + (long)i);
        return SPC_OK;
    }
    return spc::set_error(SPC_ERR_ARG, "pointer was not allocated by spc_comm_window_alloc");
}

// In-place fp32 sum of a weight gradient across the communicator's ranks,
// enqueued on `stream` (no host synchronisation).  `nccl_comm` is an
// ncclComm_t (spc_comm_nccl(comm), or the caller's own communicator).
spc_status spc_bww_allreduce(void* nccl_comm, float* dG, size_t n, void* stream) {
    if (!nccl_comm || (!dG && n)) return spc::set_error(SPC_ERR_ARG, "null comm or buffer");
    if (spc_status s = need_nccl()) return s;
    if (n == 0) return SPC_OK;
    if (ncclResult_t r = nccl().AllReduce(dG, dG, n, ncclFloat32, ncclSum, nccl_comm, (cudaStream_t)stream))
        return nccl_fail(r, "ncclAllReduce");
    return SPC_OK;
}

// BWW over this rank's batch shard, then the dG allreduce on the same stream:
// `shard_shape` carries the local N; on return (stream order) dst holds the
// dG of the global batch on every rank.  d_counters (optional) are summed
// across ranks too, so executed_vector_fmas equals the global batch's count.
spc_status spc_bww_sharded(spc_comm* comm, const spc_tensor* input, const spc_tensor* grad_out,
                           const spc_shape* shard_shape, const spc_plan* plan, int mode, spc_tensor* dst,
                           spc_counters* d_counters, void* stream) {
    if (!comm) return spc::set_error(SPC_ERR_ARG, "null comm");
    if (spc_status s = need_nccl()) return s;
    if (spc_status s = spc_sparse_bww(input, grad_out, shard_shape, plan, mode, dst, d_counters, stream)) return s;
    if (spc_status s = spc_bww_allreduce(comm->nc, static_cast<float*>(dst->data), dst->numel, stream)) return s;
    if (d_counters && comm->nranks > 1) {
        if (ncclResult_t r = nccl().AllReduce(d_counters, d_counters, 4, ncclUint64, ncclSum, comm->nc,
                                              (cudaStream_t)stream))
            return nccl_fail(r, "ncclAllReduce(counters)");
    }
    return SPC_OK;
}

}  // extern "C"

// comm.cu -- the multi-GPU exchange of SURVEY §8(e) (a13) inside the library:
// an NCCL communicator per context, the in-place allreduce of the CG scalars
// (p.q, r.z) and the grouped point-to-point halo exchange of owned rows to the
// ranks that hold them as ghosts.  All calls are stream-ordered (no host
// synchronisation), so a distributed PCG iteration is a sequence of library
// kernels and NCCL calls on one stream (CUDA-graph capturable).
//
// libnccl.so.2 is opened at run time (dlopen): the process uses the NCCL that
// is already loaded (PyTorch's) and the library has no link-time dependency.
#include <dlfcn.h>

#include <cstring>

#include "ebb_internal.cuh"

namespace ebb {
namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSum_ = 0 };
enum { ncclUint8_ = 1, ncclFloat64_ = 8 };

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
        // RTLD_NOLOAD first: prefer the copy the process already uses
        n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!n.h) n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (n.h) break;
    }
    if (!n.h) return n;
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
    n.Send = (decltype(n.Send))sym("ncclSend");
    n.Recv = (decltype(n.Recv))sym("ncclRecv");
    n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce && n.Send && n.Recv && n.GroupStart &&
           n.GroupEnd;
    return n;
}

ebb_status nccl_fail(Ctx* c, ncclResult_t r, const char* what) {
    Nccl& n = nccl();
    return fail(c, EBB_E_NCCL, "%s: NCCL error %d (%s)", what, r, n.GetErrorString ? n.GetErrorString(r) : "?");
}

}  // namespace

void comm_release(Ctx* c) {
    if (c->comm) {
        Nccl& n = nccl();
        if (n.ok) n.CommDestroy((ncclComm_t)c->comm);
        c->comm = nullptr;
    }
}

}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_comm_unique_id(ebb_nccl_id* out) {
    if (!out) return EBB_E_ARG;
    Nccl& n = nccl();
    if (!n.ok) return EBB_E_NCCL;
    ncclUniqueId id;
    if (n.GetUniqueId(&id) != 0) return EBB_E_NCCL;
    static_assert(sizeof(id) == sizeof(out->internal), "NCCL unique id size");
    memcpy(out->internal, id.internal, sizeof(id.internal));
    return EBB_OK;
}

ebb_status ebb_comm_init(ebb_ctx ctx, int32_t nranks, int32_t rank, const ebb_nccl_id* id) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !id) return fail(c, EBB_E_ARG, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, EBB_E_ARG, "comm_init: rank %d of %d", rank, nranks);
    Nccl& n = nccl();
    if (!n.ok) return fail(c, EBB_E_NCCL, "comm_init: libnccl.so.2 not found");
    comm_release(c);
    EBB_CUDA(c, cudaSetDevice(c->device));
    ncclUniqueId uid;
    memcpy(uid.internal, id->internal, sizeof(uid.internal));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = n.CommInitRank(&comm, nranks, uid, rank);
    if (r != 0) return nccl_fail(c, r, "ncclCommInitRank");
    c->comm = comm;
    c->comm_size = nranks;
    c->comm_rank = rank;
    return EBB_OK;
}

ebb_status ebb_comm_allreduce_sum(ebb_ctx ctx, double* dev_buf, uint64_t count, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !dev_buf) return fail(c, EBB_E_ARG, "null argument");
    if (!c->comm) return fail(c, EBB_E_STATE, "comm_allreduce: ebb_comm_init first");
    const ncclResult_t r = nccl().AllReduce(dev_buf, dev_buf, count, ncclFloat64_, ncclSum_, (ncclComm_t)c->comm,
                                            (cudaStream_t)s);
    if (r != 0) return nccl_fail(c, r, "ncclAllReduce");
    return EBB_OK;
}

ebb_status ebb_comm_halo(ebb_ctx ctx, int32_t npeers, const int32_t* peers, void* const* send_bufs,
                         const uint64_t* send_bytes, void* const* recv_bufs, const uint64_t* recv_bytes,
                         ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || (npeers > 0 && (!peers || !send_bufs || !send_bytes || !recv_bufs || !recv_bytes)))
        return fail(c, EBB_E_ARG, "null argument");
    if (!c->comm) return fail(c, EBB_E_STATE, "comm_halo: ebb_comm_init first");
    Nccl& n = nccl();
    ncclResult_t r = n.GroupStart();
    if (r != 0) return nccl_fail(c, r, "ncclGroupStart");
    for (int32_t k = 0; k < npeers; ++k) {
        if (peers[k] < 0 || peers[k] >= c->comm_size || peers[k] == c->comm_rank) {
            n.GroupEnd();
            return fail(c, EBB_E_ARG, "comm_halo: bad peer %d", peers[k]);
        }
        if (send_bytes[k]) {
            r = n.Send(send_bufs[k], send_bytes[k], ncclUint8_, peers[k], (ncclComm_t)c->comm, (cudaStream_t)s);
            if (r != 0) break;
        }
        if (recv_bytes[k]) {
            r = n.Recv(recv_bufs[k], recv_bytes[k], ncclUint8_, peers[k], (ncclComm_t)c->comm, (cudaStream_t)s);
            if (r != 0) break;
        }
    }
    const ncclResult_t r2 = n.GroupEnd();
    if (r != 0) return nccl_fail(c, r, "ncclSend/ncclRecv");
    if (r2 != 0) return nccl_fail(c, r2, "ncclGroupEnd");
    return EBB_OK;
}

}  // extern "C"

// collectives.cu -- NCCL inside the library, on the context stream.
//
// The multi-GPU data plane: the text broadcast from rank 0
// and the all-gather of the per-shard tie totals run as NCCL collectives on
// the library's own stream, between the library's own device buffers -- no
// torch tensors, no host round trip for the text.  torch.distributed (or any
// other channel) is needed only to hand the 128-byte ncclUniqueId from rank 0
// to the others (rs_nccl_unique_id -> rs_nccl_init).
//
// libnccl.so.2 is resolved at run time (dlopen / dlsym; nccl.h supplies the
// types only): a process that already loaded NCCL (e.g. torch's bundled copy,
// which torch.distributed brings in first) keeps using that one instead of
// mixing two NCCL builds; otherwise the system library is loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace rsb {

namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.broadcast = (decltype(a.broadcast))dlsym(h, "ncclBroadcast");
        a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
        a.errorString = (decltype(a.errorString))dlsym(h, "ncclGetErrorString");
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.broadcast && a.allGather && a.errorString;
    });
    if (!a.ok) fail(RS_ENCCL, "libnccl.so.2 not available");
    return a;
}

void check(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return;
    fail(RS_ENCCL, std::string(what) + ": " + api().errorString(r));
}

ncclComm_t comm_of(rs_ctx *c) {
    if (!c->nccl_comm) fail(RS_ESTATE, "no NCCL communicator (rs_nccl_init)");
    return (ncclComm_t)c->nccl_comm;
}

}  // namespace

void nccl_unique_id(unsigned char *out) {
    ncclUniqueId id;
    check(api().getUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id.internal) == NCCL_UNIQUE_ID_BYTES, "id size");
    std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

void nccl_init(rs_ctx *c, const unsigned char *id_bytes, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) fail(RS_EINVAL, "bad NCCL rank / world size");
    if (c->nccl_comm) {
        check(api().commDestroy((ncclComm_t)c->nccl_comm), "ncclCommDestroy");
        c->nccl_comm = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm;
    check(api().commInitRank(&comm, world, id, rank), "ncclCommInitRank");
    c->nccl_comm = comm;
    c->nccl_rank = rank;
    c->nccl_world = world;
}

void nccl_destroy(rs_ctx *c) {
    if (!c->nccl_comm) return;
    ncclResult_t r = api().commDestroy((ncclComm_t)c->nccl_comm);
    c->nccl_comm = nullptr;
    check(r, "ncclCommDestroy");
}

// text bytes [0, n) of B_TEXT from `root` to every rank (in place)
void nccl_broadcast_text(rs_ctx *c, long long n, int root) {
    unsigned char *d = (unsigned char *)buf(c, B_TEXT, (size_t)n + 128);
    if (n > 0) check(api().broadcast(d, d, (size_t)n, ncclUint8, root, comm_of(c), c->stream), "ncclBroadcast");
    RS_CUDA(cudaMemsetAsync(d + n, 0, 128, c->stream));
    RS_CUDA(cudaStreamSynchronize(c->stream));
}

// one int64 per rank -> every rank's values, rank order
void nccl_allgather_i64(rs_ctx *c, long long value, long long *out) {
    const int world = c->nccl_world;
    long long *d = (long long *)((char *)buf(c, B_SMALL, 4096) + 1024);
    if (world > 256) fail(RS_EINVAL, "world size above 256");
    RS_CUDA(cudaMemcpyAsync(d, &value, sizeof(value), cudaMemcpyHostToDevice, c->stream));
    check(api().allGather(d, d + 1, 1, ncclInt64, comm_of(c), c->stream), "ncclAllGather");
    RS_CUDA(cudaMemcpyAsync(out, d + 1, sizeof(long long) * (size_t)world, cudaMemcpyDeviceToHost, c->stream));
    RS_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace rsb

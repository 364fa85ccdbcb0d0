// comm.cpp — row a9 of SURVEY §8: the cross-GPU exchange over NCCL (NVLink 5 / NVSwitch).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") so that libgalois loads
// without it and shares the copy torch already mapped into the process (no second NCCL).
// The engine uses three collectives: an 8-byte MIN all-reduce of the best key per check
// interval, an n-byte broadcast of the winner's bits when queried, and nothing else (the
// batch members share no parameters, so there is no gradient exchange).
#include "comm.h"

#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <mutex>

namespace galois {

namespace {

struct NcclApi {
    bool tried = false;
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_api;
std::mutex g_mu;

template <typename F>
bool sym(void *h, const char *name, F &out)
{
    out = reinterpret_cast<F>(dlsym(h, name));
    return out != nullptr;
}

}  // namespace

bool nccl_load(std::string *why)
{
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_api.tried) {
        g_api.tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            g_api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
        } else if (!sym(h, "ncclGetUniqueId", g_api.GetUniqueId) ||
                   !sym(h, "ncclCommInitRank", g_api.CommInitRank) ||
                   !sym(h, "ncclCommDestroy", g_api.CommDestroy) ||
                   !sym(h, "ncclCommAbort", g_api.CommAbort) ||
                   !sym(h, "ncclAllReduce", g_api.AllReduce) ||
                   !sym(h, "ncclBroadcast", g_api.Broadcast) ||
                   !sym(h, "ncclGetErrorString", g_api.GetErrorString)) {
            g_api.why = "libnccl.so.2 lacks a required symbol";
        } else {
            g_api.ok = true;
        }
    }
    if (!g_api.ok && why) *why = g_api.why;
    return g_api.ok;
}

static std::string nccl_err(const char *what, ncclResult_t r)
{
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, g_api.GetErrorString ? g_api.GetErrorString(r) : "nccl error");
    return buf;
}

bool nccl_unique_id(void *out128, std::string *why)
{
    if (!nccl_load(why)) return false;
    ncclUniqueId id;
    ncclResult_t r = g_api.GetUniqueId(&id);
    if (r != ncclSuccess) {
        if (why) *why = nccl_err("ncclGetUniqueId", r);
        return false;
    }
    memcpy(out128, &id, sizeof(id));
    return true;
}

bool Comm::init(int rank_, int world_, const unsigned char *id128, std::string *why)
{
    rank = rank_;
    world = world_;
    if (!nccl_load(why)) return false;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclResult_t r = g_api.CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) {
        comm = nullptr;
        if (why) *why = nccl_err("ncclCommInitRank", r);
        return false;
    }
    return true;
}

bool Comm::allreduce_min_u64(const unsigned long long *send, unsigned long long *recv, cudaStream_t st,
                             std::string *why)
{
    ncclResult_t r = g_api.AllReduce(send, recv, 1, ncclUint64, ncclMin, comm, st);
    if (r != ncclSuccess) {
        if (why) *why = nccl_err("ncclAllReduce", r);
        return false;
    }
    return true;
}

bool Comm::broadcast_bytes(void *buf, size_t bytes, int root, cudaStream_t st, std::string *why)
{
    ncclResult_t r = g_api.Broadcast(buf, buf, bytes, ncclUint8, root, comm, st);
    if (r != ncclSuccess) {
        if (why) *why = nccl_err("ncclBroadcast", r);
        return false;
    }
    return true;
}

void Comm::destroy(bool abort)
{
    if (comm) {
        if (abort) g_api.CommAbort(comm); else g_api.CommDestroy(comm);
        comm = nullptr;
    }
}

}  // namespace galois

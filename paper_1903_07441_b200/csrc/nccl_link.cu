// nccl_link.cu -- the NCCL calls of row-slab contexts: ghost-row send/recv, the
// residual max all-reduce and the walker hand-over broadcast, plus the communicator helpers of the
// C ABI (twg_nccl_unique_id / twg_nccl_comm_init / twg_nccl_comm_destroy).
//
// libtwg does not link NCCL: the entry points are resolved at run time from the libnccl.so.2 the
// process already has loaded (torch's, so a communicator made by torch and one made here are the
// same library), else from libnccl.so.2 by name (or $TWG_NCCL_LIB).  Only the stable C ABI of
// nccl.h 2.x is used; the few types are declared here.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "api_host.cuh"

namespace twg {
namespace host {
namespace {

typedef void* ncclComm_t;
typedef int ncclResult_t;  // ncclSuccess = 0
struct ncclUniqueId {
    char internal[128];
};
enum { kNcclInt32 = 2, kNcclUint32 = 3, kNcclFloat32 = 7 };
enum { kNcclMax = 2 };

struct Fns {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commCount)(ncclComm_t, int*) = nullptr;
    ncclResult_t (*commUserRank)(ncclComm_t, int*) = nullptr;
    ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string err;
};

Fns g_fns;
std::once_flag g_once;

void load_once() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy the process already uses
    if (!h) {
        const char* env = std::getenv("TWG_NCCL_LIB");
        if (env && env[0]) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_fns.err = std::string("libnccl.so.2 not found: ") + dlerror();
        return;
    }
    bool ok = true;
    auto get = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        if (!fp) {
            ok = false;
            g_fns.err = std::string("libnccl.so.2 lacks ") + name;
        }
    };
    get(g_fns.getUniqueId, "ncclGetUniqueId");
    get(g_fns.commInitRank, "ncclCommInitRank");
    get(g_fns.commDestroy, "ncclCommDestroy");
    get(g_fns.commCount, "ncclCommCount");
    get(g_fns.commUserRank, "ncclCommUserRank");
    get(g_fns.send, "ncclSend");
    get(g_fns.recv, "ncclRecv");
    get(g_fns.allReduce, "ncclAllReduce");
    get(g_fns.broadcast, "ncclBroadcast");
    get(g_fns.groupStart, "ncclGroupStart");
    get(g_fns.groupEnd, "ncclGroupEnd");
    get(g_fns.errorString, "ncclGetErrorString");
    g_fns.ok = ok;
}

bool loaded(std::string* why) {
    std::call_once(g_once, load_once);
    if (!g_fns.ok && why) *why = g_fns.err;
    return g_fns.ok;
}

}  // namespace

#define TWG_NCCL(ctx, expr)                                                                              \
    do {                                                                                                 \
        ncclResult_t r_ = (expr);                                                                        \
        if (r_ != 0) return fail(ctx, TWG_E_NCCL, std::string(#expr) + ": " + g_fns.errorString(r_));     \
    } while (0)

twg_status nccl_load(twg_ctx* c) {
    std::string why;
    if (!loaded(&why)) return fail(c, TWG_E_NCCL, why);
    return TWG_OK;
}

twg_status nccl_comm_rank(twg_ctx* c, void* comm, int* rank, int* nranks) {
    twg_status st = nccl_load(c);
    if (st != TWG_OK) return st;
    TWG_NCCL(c, g_fns.commUserRank(comm, rank));
    TWG_NCCL(c, g_fns.commCount(comm, nranks));
    return TWG_OK;
}

twg_status nccl_exchange(twg_ctx* c, size_t cnt, int up, int dn, const float* s_up, float* r_up, const float* s_dn,
                         float* r_dn, cudaStream_t st) {
    ncclComm_t comm = c->shard.nccl;
    TWG_NCCL(c, g_fns.groupStart());
    if (up >= 0) {
        TWG_NCCL(c, g_fns.send(s_up, cnt, kNcclFloat32, up, comm, st));
        TWG_NCCL(c, g_fns.recv(r_up, cnt, kNcclFloat32, up, comm, st));
    }
    if (dn >= 0) {
        TWG_NCCL(c, g_fns.send(s_dn, cnt, kNcclFloat32, dn, comm, st));
        TWG_NCCL(c, g_fns.recv(r_dn, cnt, kNcclFloat32, dn, comm, st));
    }
    TWG_NCCL(c, g_fns.groupEnd());
    return TWG_OK;
}

twg_status nccl_allreduce_max_u32(twg_ctx* c, unsigned* buf, int n, cudaStream_t st) {
    TWG_NCCL(c, g_fns.allReduce(buf, buf, (size_t)n, kNcclUint32, kNcclMax, c->shard.nccl, st));
    return TWG_OK;
}

twg_status nccl_allreduce_sum_u32(twg_ctx* c, unsigned* buf, size_t n, cudaStream_t st) {
    TWG_NCCL(c, g_fns.allReduce(buf, buf, n, kNcclUint32, 0 /* ncclSum */, c->shard.nccl, st));
    return TWG_OK;
}

twg_status nccl_bcast_i32(twg_ctx* c, int* buf, int n, int root, cudaStream_t st) {
    TWG_NCCL(c, g_fns.broadcast(buf, buf, (size_t)n, kNcclInt32, root, c->shard.nccl, st));
    return TWG_OK;
}

}  // namespace host
}  // namespace twg

using namespace twg::host;

TWG_API twg_status twg_nccl_unique_id(void* out, int32_t bytes) {
    std::string why;
    if (!out || bytes < (int32_t)sizeof(ncclUniqueId)) return fail(nullptr, TWG_E_INVALID_ARG, "id buffer < 128 bytes");
    if (!loaded(&why)) return fail(nullptr, TWG_E_NCCL, why);
    ncclUniqueId id;
    ncclResult_t r = g_fns.getUniqueId(&id);
    if (r != 0) return fail(nullptr, TWG_E_NCCL, std::string("ncclGetUniqueId: ") + g_fns.errorString(r));
    std::memcpy(out, &id, sizeof(id));
    return TWG_OK;
}

TWG_API twg_status twg_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, int32_t device, void** comm) {
    std::string why;
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, TWG_E_INVALID_ARG, "bad argument");
    if (!loaded(&why)) return fail(nullptr, TWG_E_NCCL, why);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(nullptr, TWG_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t cm = nullptr;
    ncclResult_t r = g_fns.commInitRank(&cm, nranks, u, rank);
    if (r != 0) return fail(nullptr, TWG_E_NCCL, std::string("ncclCommInitRank: ") + g_fns.errorString(r));
    *comm = cm;
    return TWG_OK;
}

TWG_API twg_status twg_nccl_comm_destroy(void* comm) {
    std::string why;
    if (!comm) return TWG_OK;
    if (!loaded(&why)) return fail(nullptr, TWG_E_NCCL, why);
    ncclResult_t r = g_fns.commDestroy(comm);
    if (r != 0) return fail(nullptr, TWG_E_NCCL, std::string("ncclCommDestroy: ") + g_fns.errorString(r));
    return TWG_OK;
}

// comm.cpp -- dlopen'd NCCL transport (see comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

namespace mpj {

namespace {

struct NcclApi {
    bool ok = false;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclBroadcast) Broadcast = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommGetAsyncError) GetAsyncError = nullptr;
};

NcclApi g_api;
std::once_flag g_once;
char g_err[256] = "no error";

void load_api() {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* nm : names) {
        h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        snprintf(g_err, sizeof(g_err), "dlopen(libnccl.so.2) failed: %s", dlerror());
        return;
    }
#define MPJ_SYM(field, sym)                                                   \
    g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, #sym));   \
    if (!g_api.field) {                                                       \
        snprintf(g_err, sizeof(g_err), "NCCL symbol %s missing", #sym);       \
        return;                                                               \
    }
    MPJ_SYM(GetUniqueId, ncclGetUniqueId)
    MPJ_SYM(CommInitRank, ncclCommInitRank)
    MPJ_SYM(CommDestroy, ncclCommDestroy)
    MPJ_SYM(GroupStart, ncclGroupStart)
    MPJ_SYM(GroupEnd, ncclGroupEnd)
    MPJ_SYM(Send, ncclSend)
    MPJ_SYM(Recv, ncclRecv)
    MPJ_SYM(Broadcast, ncclBroadcast)
    MPJ_SYM(AllReduce, ncclAllReduce)
    MPJ_SYM(GetErrorString, ncclGetErrorString)
    MPJ_SYM(GetAsyncError, ncclCommGetAsyncError)
#undef MPJ_SYM
    g_api.ok = true;
}

const NcclApi* api() {
    std::call_once(g_once, load_api);
    return g_api.ok ? &g_api : nullptr;
}

constexpr int ERR_NCCL = -5;

int check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return 0;
    snprintf(g_err, sizeof(g_err), "%s: %s", what, g_api.GetErrorString ? g_api.GetErrorString(r) : "?");
    return ERR_NCCL;
}

}  // namespace

const char* nccl_last_error() { return g_err; }

int nccl_unique_id(unsigned char* out) {
    const NcclApi* a = api();
    if (!a) return ERR_NCCL;
    ncclUniqueId id;
    int rc = check(a->GetUniqueId(&id), "ncclGetUniqueId");
    if (rc) return rc;
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return 0;
}

int Comm::init(int rank_, int world_, const unsigned char* id) {
    const NcclApi* a = api();
    if (!a) return ERR_NCCL;
    destroy();
    ncclUniqueId uid;
    memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    int rc = check(a->CommInitRank(&c, world_, uid, rank_), "ncclCommInitRank");
    if (rc) return rc;
    comm_ = c;
    rank = rank_;
    world = world_;
    return 0;
}

void Comm::destroy() {
    if (comm_ && g_api.ok) g_api.CommDestroy(static_cast<ncclComm_t>(comm_));
    comm_ = nullptr;
    rank = 0;
    world = 1;
}

int Comm::bcast(void* buf, size_t bytes, int root, cudaStream_t st) {
    return check(g_api.Broadcast(buf, buf, bytes, ncclInt8, root, static_cast<ncclComm_t>(comm_), st),
                 "ncclBroadcast");
}
int Comm::group_start() { return check(g_api.GroupStart(), "ncclGroupStart"); }
int Comm::group_end() { return check(g_api.GroupEnd(), "ncclGroupEnd"); }
int Comm::send(const void* buf, size_t bytes, int peer, cudaStream_t st) {
    return check(g_api.Send(buf, bytes, ncclInt8, peer, static_cast<ncclComm_t>(comm_), st), "ncclSend");
}
int Comm::recv(void* buf, size_t bytes, int peer, cudaStream_t st) {
    return check(g_api.Recv(buf, bytes, ncclInt8, peer, static_cast<ncclComm_t>(comm_), st), "ncclRecv");
}
int Comm::allreduce_max_f64(double* buf, size_t count, cudaStream_t st) {
    return check(g_api.AllReduce(buf, buf, count, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm_), st),
                 "ncclAllReduce(max)");
}
int Comm::allreduce_max_i64(long long* buf, size_t count, cudaStream_t st) {
    return check(g_api.AllReduce(buf, buf, count, ncclInt64, ncclMax, static_cast<ncclComm_t>(comm_), st),
                 "ncclAllReduce(max)");
}
int Comm::async_error() {
    if (!comm_) return 0;
    ncclResult_t ae = ncclSuccess;
    int rc = check(g_api.GetAsyncError(static_cast<ncclComm_t>(comm_), &ae), "ncclCommGetAsyncError");
    if (rc) return rc;
    return check(ae, "NCCL asynchronous error");
}

int Comm::allreduce_sum_i32(int* buf, size_t count, cudaStream_t st) {
    return check(g_api.AllReduce(buf, buf, count, ncclInt32, ncclSum, static_cast<ncclComm_t>(comm_), st),
                 "ncclAllReduce(sum)");
}

}  // namespace mpj

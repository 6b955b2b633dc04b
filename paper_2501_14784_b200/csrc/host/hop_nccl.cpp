// NCCL resolution and ring-link setup (see hop_nccl.hpp).
#include "hop_nccl.hpp"

#include <dlfcn.h>

#include <mutex>

#include "pipeline.hpp"

namespace dsb {

const NcclApi* nccl_api(std::string* why) {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        if (!api.GetUniqueId || !api.CommInitRank || !api.Recv || !api.GroupStart || !api.GroupEnd) {
            api.Send = nullptr;
            api.error = "libnccl is missing point-to-point symbols";
        }
    });
    if (!api.ok()) {
        if (why) *why = api.error;
        return nullptr;
    }
    return &api;
}

void RingLinks::init(const NcclApi& api, int rank, int world, const ncclUniqueId* ids) {
    auto chk = [&](ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw SimError(std::string(what) + ": " + api.GetErrorString(r));
    };
    const int prev = (rank + world - 1) % world;
    rank_ = rank;
    world_ = world;
    chk(api.GroupStart(), "ncclGroupStart");
    chk(api.CommInitRank(&send, 2, ids[rank], 0), "ncclCommInitRank(send link)");
    chk(api.CommInitRank(&recv, 2, ids[prev], 1), "ncclCommInitRank(recv link)");
    chk(api.GroupEnd(), "ncclGroupEnd");
}

void RingLinks::warmup(const NcclApi& api, void* send_buf, void* recv_buf, cudaStream_t stream) {
    auto chk = [&](ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw SimError(std::string(what) + ": " + api.GetErrorString(r));
    };
    chk(api.GroupStart(), "ncclGroupStart");
    chk(api.Send(send_buf, 16, ncclUint8, 1, send, stream), "ncclSend(warmup)");
    chk(api.Recv(recv_buf, 16, ncclUint8, 0, recv, stream), "ncclRecv(warmup)");
    chk(api.GroupEnd(), "ncclGroupEnd");
}

// ncclCommDestroy finalizes with the peer, so every rank tears its two links down in global
// link-index order (link i joins ranks i and i+1): the wait graph stays acyclic.
void RingLinks::destroy(const NcclApi& api) {
    const int send_link = rank_, recv_link = (rank_ + world_ - 1) % world_;
    ncclComm_t first = send_link < recv_link ? send : recv;
    ncclComm_t second = send_link < recv_link ? recv : send;
    if (first) api.CommDestroy(first);
    if (second) api.CommDestroy(second);
    send = recv = nullptr;
}

void RingLinks::abort(const NcclApi& api) {
    if (api.CommAbort) {
        if (send) api.CommAbort(send);
        if (recv) api.CommAbort(recv);
    }
    send = recv = nullptr;
}

}  // namespace dsb

// Stage-to-stage hops over NCCL point-to-point (one process per GPU). The ring i -> i+1 uses one
// 2-rank communicator per link so a rank's sends (its link) and receives (the previous rank's
// link) progress on independent communicators and streams: a ring of blocking sends can never
// wait on a receive queued behind it. libnccl is resolved at run time (dlopen "libnccl.so.2"), so
// the library loads on hosts without NCCL and shares torch's copy when one is already loaded.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace dsb {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
    bool ok() const { return Send != nullptr; }
};

// Loads libnccl once; returns nullptr (with a message) if unavailable.
const NcclApi* nccl_api(std::string* why);

// Per-rank hop endpoints: send = link rank -> rank+1 (this rank is comm rank 0), recv = link
// rank-1 -> rank (this rank is comm rank 1). ids: world unique ids, one per link.
struct RingLinks {
    ncclComm_t send = nullptr, recv = nullptr;
    void init(const NcclApi& api, int rank, int world, const ncclUniqueId* ids);
    // one tiny send on the send link and receive on the recv link, grouped: establishes both
    // p2p connections on every rank at once
    void warmup(const NcclApi& api, void* send_buf, void* recv_buf, cudaStream_t stream);
    void destroy(const NcclApi& api);
    // failure path: abort both communicators (pending sends / receives return, no finalize
    // handshake with a peer that may be gone)
    void abort(const NcclApi& api);
    int rank_ = 0, world_ = 1;
};

}  // namespace dsb

#include "comm.hpp"

#include <cstring>

#include "common.cuh"

namespace flw {

std::string Comm::new_unique_id() {
    ncclUniqueId id;
    FLW_NCCL(ncclGetUniqueId(&id));
    return std::string(id.internal, sizeof(id.internal));
}

Comm::Comm(const std::string& unique_id, int rank, int nranks, int device) : rank_(rank), nranks_(nranks) {
    if (unique_id.size() != sizeof(ncclUniqueId::internal)) fail(Errc::Config, "bad NCCL unique id length");
    ncclUniqueId id;
    std::memcpy(id.internal, unique_id.data(), sizeof(id.internal));
    if (cudaSetDevice(device) != cudaSuccess) fail(Errc::Runtime, "cudaSetDevice failed for NCCL init");
    FLW_NCCL(ncclCommInitRank(&comm_, nranks, id, rank));
}

std::vector<ncclComm_t> Comm::init_all(const std::vector<int>& devices) {
    std::vector<ncclComm_t> comms(devices.size());
    flw_trace("nccl init_all");
    FLW_NCCL(ncclCommInitAll(comms.data(), static_cast<int>(devices.size()), devices.data()));
    return comms;
}

void Comm::connect_all(const std::vector<Comm*>& comms, const std::vector<int>& devices, int64_t count) {
    // Eager grouped collectives of the real sizes (the gradient all-gather and all-reduce), so
    // every peer connection and protocol buffer exists before any rank captures its
    // collectives into a CUDA graph from its own thread.
    const size_t k = comms.size();
    std::vector<float*> buf(k, nullptr);
    std::vector<cudaStream_t> st(k, nullptr);
    for (size_t r = 0; r < k; ++r) {
        FLW_CUDA(cudaSetDevice(devices[r]));
        FLW_CUDA(cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking));
        FLW_CUDA(cudaMalloc(&buf[r], sizeof(float) * static_cast<size_t>(count) * (k + 1)));
        FLW_CUDA(cudaMemset(buf[r], 0, sizeof(float) * static_cast<size_t>(count) * (k + 1)));
    }
    flw_trace("nccl connect: all_gather");
    FLW_NCCL(ncclGroupStart());
    for (size_t r = 0; r < k; ++r)
        FLW_NCCL(ncclAllGather(buf[r], buf[r] + count, static_cast<size_t>(count), ncclFloat32, comms[r]->comm_, st[r]));
    FLW_NCCL(ncclGroupEnd());
    flw_trace("nccl connect: all_reduce");
    FLW_NCCL(ncclGroupStart());
    for (size_t r = 0; r < k; ++r)
        FLW_NCCL(ncclAllReduce(buf[r], buf[r], static_cast<size_t>(count), ncclFloat32, ncclSum, comms[r]->comm_, st[r]));
    FLW_NCCL(ncclGroupEnd());
    for (size_t r = 0; r < k; ++r) {
        FLW_CUDA(cudaSetDevice(devices[r]));
        FLW_CUDA(cudaStreamSynchronize(st[r]));
        FLW_CUDA(cudaStreamDestroy(st[r]));
        FLW_CUDA(cudaFree(buf[r]));
    }
    flw_trace("nccl connect: done");
}

Comm::~Comm() {
    if (comm_) {
        if (aborted_) return;  // ncclCommAbort already released it
        ncclCommDestroy(comm_);
    }
}

void Comm::abort() {
    // Unblocks peers whose collective kernels wait for a rank that failed (the reference's
    // PeerFailure path, local_run.cpp:536-548): every rank's comm is aborted, not destroyed.
    if (comm_ && !aborted_.exchange(true)) ncclCommAbort(comm_);
}

void Comm::all_gather(const float* send, float* recv, int64_t count, cudaStream_t s) {
    FLW_NCCL(ncclAllGather(send, recv, static_cast<size_t>(count), ncclFloat32, comm_, s));
}

void Comm::all_reduce_sum(const float* send, float* recv, int64_t count, cudaStream_t s) {
    FLW_NCCL(ncclAllReduce(send, recv, static_cast<size_t>(count), ncclFloat32, ncclSum, comm_, s));
}

}  // namespace flw

#include "comm.hpp"

#include <cstring>

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
    FLW_NCCL(ncclCommInitAll(comms.data(), static_cast<int>(devices.size()), devices.data()));
    return comms;
}

Comm::~Comm() {
    if (comm_) ncclCommDestroy(comm_);
}

void Comm::all_gather(const float* send, float* recv, int64_t count, cudaStream_t s) {
    FLW_NCCL(ncclAllGather(send, recv, static_cast<size_t>(count), ncclFloat32, comm_, s));
}

void Comm::all_reduce_sum(const float* send, float* recv, int64_t count, cudaStream_t s) {
    FLW_NCCL(ncclAllReduce(send, recv, static_cast<size_t>(count), ncclFloat32, ncclSum, comm_, s));
}

}  // namespace flw

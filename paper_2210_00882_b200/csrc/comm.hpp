// Gradient group over NCCL (NVLink 5 / NVSwitch on one node): the B200 replacement for the
// reference's GradSync mailbox AllGather (local_run.cpp:379-414, channels.cpp:9-41).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "errors.hpp"

namespace flw {

#define FLW_NCCL(x)                                                                                   \
    do {                                                                                              \
        ncclResult_t r_ = (x);                                                                        \
        if (r_ != ncclSuccess)                                                                        \
            throw ::flw::Error(::flw::Errc::PeerFailure, std::string("NCCL: ") + ncclGetErrorString(r_)); \
    } while (0)

class Comm {
  public:
    // One rank of a group whose unique id was produced by new_unique_id() on rank 0 and
    // distributed out of band (torch.distributed store in multi-process runs).
    Comm(const std::string& unique_id, int rank, int nranks, int device);
    // Adopt a communicator created by ncclCommInitAll (single-process, one thread per GPU).
    Comm(ncclComm_t comm, int rank, int nranks) : comm_(comm), rank_(rank), nranks_(nranks) {}
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;

    static std::string new_unique_id();  // NCCL_UNIQUE_ID_BYTES raw bytes
    static std::vector<ncclComm_t> init_all(const std::vector<int>& devices);
    static void connect_all(const std::vector<Comm*>& comms, const std::vector<int>& devices, int64_t count);

    void all_gather(const float* send, float* recv, int64_t count, cudaStream_t s);
    void all_reduce_sum(const float* send, float* recv, int64_t count, cudaStream_t s);
    void abort();
    int rank() const { return rank_; }
    int nranks() const { return nranks_; }

  private:
    ncclComm_t comm_ = nullptr;
    std::atomic<bool> aborted_{false};
    int rank_ = 0, nranks_ = 1;
};

}  // namespace flw

// Point-to-point transports of the multi-GPU (mesh-partitioned) schedule: NCCL send/recv over
// NVLink between processes (libnccl resolved at run time, so the library loads without it), and
// an in-process loopback (buffered sends through a shared hub, blocking receives) that lets two
// contexts on one device play two ranks from two host threads -- the single-GPU test of the
// partition and exchange logic.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <string>

namespace mrab {

struct Transport {
    virtual ~Transport() {}
    // begin / end bracket the sends and receives of one exchange (an NCCL group)
    virtual bool begin() = 0;
    virtual bool send(const void* dev, size_t bytes, int peer, int tag, cudaStream_t st) = 0;
    virtual bool recv(void* dev, size_t bytes, int peer, int tag, cudaStream_t st) = 0;
    virtual bool end(cudaStream_t st) = 0;
    std::string err;
};

// NCCL: `unique_id` = the 128-byte ncclUniqueId of the job (from nccl_unique_id on rank 0)
std::unique_ptr<Transport> make_nccl_transport(const void* unique_id, int rank, int nranks, std::string* err);
bool nccl_unique_id(void* out128, std::string* err);
// loopback: every context attached with the same world id shares one hub
std::unique_ptr<Transport> make_loopback_transport(int world_id, int rank, int nranks);

}  // namespace mrab

// comm.h -- inter-GPU plumbing of libhetpipe for the distributed placements:
// a stream-ordered barrier among the ranks (NCCL all-reduce of one int, loaded
// with dlopen so the library uses the NCCL the process already has) and CUDA
// IPC for mapping every peer's arena (one process per GPU).
//
// The data itself never goes through NCCL: the tick kernels read remote acc
// slices (push) and remote w_global shards (pull) through the mapped peer
// pointers over NVLink; the barrier only orders those reads against the
// producers (PAPER.md P:928-930 push/apply, P:949 pull).
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace hp {

constexpr int kCommIdBytes = 128;   // = NCCL_UNIQUE_ID_BYTES
constexpr int kIpcBytes = 64;       // = sizeof(cudaIpcMemHandle_t)

class Comm {
 public:
  virtual ~Comm() {}
  // Device-side barrier on `stream`: later work on the stream runs only after
  // every rank's stream reached its own barrier call. Returns 0 or an error.
  virtual int barrier(cudaStream_t stream) = 0;
  virtual std::string error() const = 0;
};

// Fresh communicator id (called on one rank, broadcast by the caller).
int comm_unique_id(void* out, std::string* err);
// Collective over all ranks (same id). nullptr on failure (err set).
Comm* comm_create(const void* id, int world, int rank, std::string* err);

}  // namespace hp

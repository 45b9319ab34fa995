// comm.h -- inter-GPU plumbing of libhetpipe for the distributed placements:
// the NCCL communicator (dlopen'd, so the library uses the NCCL the process
// already has): the set-up barrier, the fallback exchange barrier (an
// all-reduce of one int; the default is the device flag barrier of
// engine.cpp xbarrier, K7) and the NCCL transport's collectives.
//
// Under HP_XPORT_PEER / NVLS the data never goes through NCCL: the tick
// kernels read remote acc slices (push) and remote w_global shards (pull)
// through the mapped peer pointers (or the multicast mapping) over NVLink; the
// barrier only orders those accesses against the producers (PAPER.md P:928-930
// push/apply, P:949 pull). HP_XPORT_NCCL, the unfused baseline, moves lockstep
// batches with the two grouped collectives below.
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
  // Reduce-scatter with uneven shards: shard q = [b[q], b[q+1]) of every
  // rank's `send` (fp32, indexed from 0) is summed into rank q's `recv`
  // (b[q+1]-b[q] floats). One ncclReduce per shard in one group.
  virtual int reduce_scatter_v(const float* send, float* recv, const int64_t* b,
                               cudaStream_t stream) = 0;
  // All-gather with uneven shards: rank q's `send` (its shard) lands at
  // recv + b[q] on every rank. One ncclBroadcast per shard in one group.
  virtual int all_gather_v(const float* send, float* recv, const int64_t* b,
                           cudaStream_t stream) = 0;
  // The equal-count forms (ncclReduceScatter / ncclAllGather): send / recv
  // hold world x count floats (rank q's block at q x count).
  virtual int reduce_scatter(const float* send, float* recv, int64_t count,
                             cudaStream_t stream) = 0;
  virtual int all_gather(const float* send, float* recv, int64_t count, cudaStream_t stream) = 0;
  virtual std::string error() const = 0;
};

// Fresh communicator id (called on one rank, broadcast by the caller).
int comm_unique_id(void* out, std::string* err);
// Collective over all ranks (same id). nullptr on failure (err set).
Comm* comm_create(const void* id, int world, int rank, std::string* err);

}  // namespace hp

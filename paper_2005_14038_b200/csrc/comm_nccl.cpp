// comm_nccl.cpp -- Comm over NCCL (dlopen'd; the process's own libnccl.so.2,
// e.g. the one torch loaded, is reused). Only a 4-byte all-reduce is issued:
// it completes on a rank only after every rank's stream reached it, which is
// the device-side barrier the distributed flush needs.
#include <dlfcn.h>
#include <cstdlib>

#include <cstring>
#include <string>

#include "comm.h"

namespace hp {
namespace {

typedef int ncclResult_t;
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
  char internal[kCommIdBytes];
};
enum { ncclInt32 = 2, ncclFloat32 = 7, ncclSum = 0 };

struct Api {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Api* api(std::string* err) {
  static Api a;
  static bool tried = false;
  if (tried) {
    if (!a.h && err) *err = "libnccl.so.2 not loadable";
    return a.h ? &a : nullptr;
  }
  tried = true;
  // the NCCL the process already has (torch loads its own), else $HP_NCCL_LIB
  // (the binding points it at torch's bundled copy), else the loader's search
  a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!a.h)
    if (const char* env = getenv("HP_NCCL_LIB")) a.h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!a.h) {
    if (err) *err = "libnccl.so.2 not loadable";
    return nullptr;
  }
  a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.h, "ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.h, "ncclCommInitRank");
  a.AllReduce = (decltype(a.AllReduce))dlsym(a.h, "ncclAllReduce");
  a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
  a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
  a.Reduce = (decltype(a.Reduce))dlsym(a.h, "ncclReduce");
  a.Broadcast = (decltype(a.Broadcast))dlsym(a.h, "ncclBroadcast");
  a.GroupStart = (decltype(a.GroupStart))dlsym(a.h, "ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))dlsym(a.h, "ncclGroupEnd");
  a.ReduceScatter = (decltype(a.ReduceScatter))dlsym(a.h, "ncclReduceScatter");
  a.AllGather = (decltype(a.AllGather))dlsym(a.h, "ncclAllGather");
  if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.CommDestroy || !a.Reduce ||
      !a.Broadcast || !a.GroupStart || !a.GroupEnd || !a.ReduceScatter || !a.AllGather) {
    a.h = nullptr;
    if (err) *err = "libnccl.so.2 lacks required symbols";
    return nullptr;
  }
  return &a;
}

class NcclComm : public Comm {
 public:
  NcclComm(Api* a, ncclComm_t c, int* scratch, int world, int rank)
      : a_(a), c_(c), scratch_(scratch), world_(world), rank_(rank) {}
  ~NcclComm() override {
    if (c_) a_->CommDestroy(c_);
    if (scratch_) cudaFree(scratch_);
  }
  int barrier(cudaStream_t s) override {
    ncclResult_t r = a_->AllReduce(scratch_, scratch_ + 1, 1, ncclInt32, ncclSum, c_, s);
    if (r != 0) err_ = a_->GetErrorString ? a_->GetErrorString(r) : "ncclAllReduce failed";
    return r;
  }
  int reduce_scatter_v(const float* send, float* recv, const int64_t* b,
                       cudaStream_t s) override {
    ncclResult_t r = a_->GroupStart();
    for (int q = 0; q < world_ && r == 0; ++q)
      r = a_->Reduce(send + b[q], q == rank_ ? recv : nullptr, (size_t)(b[q + 1] - b[q]),
                     ncclFloat32, ncclSum, q, c_, s);
    const ncclResult_t r2 = a_->GroupEnd();
    return note(r ? r : r2, "ncclReduce (reduce-scatter)");
  }
  int all_gather_v(const float* send, float* recv, const int64_t* b, cudaStream_t s) override {
    ncclResult_t r = a_->GroupStart();
    for (int q = 0; q < world_ && r == 0; ++q)
      r = a_->Broadcast(q == rank_ ? send : nullptr, recv + b[q], (size_t)(b[q + 1] - b[q]),
                        ncclFloat32, q, c_, s);
    const ncclResult_t r2 = a_->GroupEnd();
    return note(r ? r : r2, "ncclBroadcast (all-gather)");
  }
  int reduce_scatter(const float* send, float* recv, int64_t count, cudaStream_t s) override {
    return note(a_->ReduceScatter(send, recv, (size_t)count, ncclFloat32, ncclSum, c_, s),
                "ncclReduceScatter");
  }
  int all_gather(const float* send, float* recv, int64_t count, cudaStream_t s) override {
    return note(a_->AllGather(send, recv, (size_t)count, ncclFloat32, c_, s), "ncclAllGather");
  }
  std::string error() const override { return err_; }

 private:
  int note(ncclResult_t r, const char* what) {
    if (r != 0) err_ = std::string(what) + ": " + (a_->GetErrorString ? a_->GetErrorString(r) : "");
    return r;
  }
  Api* a_;
  ncclComm_t c_;
  int* scratch_;
  int world_, rank_;
  std::string err_;
};

}  // namespace

int comm_unique_id(void* out, std::string* err) {
  Api* a = api(err);
  if (!a) return -1;
  ncclUniqueId id;
  ncclResult_t r = a->GetUniqueId(&id);
  if (r != 0) {
    if (err) *err = "ncclGetUniqueId failed";
    return r;
  }
  memcpy(out, id.internal, kCommIdBytes);
  return 0;
}

Comm* comm_create(const void* id, int world, int rank, std::string* err) {
  Api* a = api(err);
  if (!a) return nullptr;
  ncclUniqueId uid;
  memcpy(uid.internal, id, kCommIdBytes);
  ncclComm_t c = nullptr;
  ncclResult_t r = a->CommInitRank(&c, world, uid, rank);
  if (r != 0) {
    if (err) *err = std::string("ncclCommInitRank: ") + (a->GetErrorString ? a->GetErrorString(r) : "");
    return nullptr;
  }
  int* scratch = nullptr;
  if (cudaMalloc(&scratch, 2 * sizeof(int)) != cudaSuccess) {
    a->CommDestroy(c);
    if (err) *err = "barrier scratch allocation failed";
    return nullptr;
  }
  cudaMemset(scratch, 0, 2 * sizeof(int));
  return new NcclComm(a, c, scratch, world, rank);
}

}  // namespace hp

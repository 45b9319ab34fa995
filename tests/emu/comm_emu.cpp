// TEST-ONLY Comm for the host emulation: ranks are threads of one process;
// the "device barrier" blocks the calling host thread until every rank of the
// same id arrives (emulated kernels run synchronously at launch, so host order
// is device order).
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../paper_2005_14038_b200/csrc/comm.h"

namespace hp {
namespace {

struct Bar {
  std::mutex mu;
  std::condition_variable cv;
  int world = 0, arrived = 0;
  long gen = 0;
  std::vector<const float*> posted;   // per rank: the send buffer of a collective
  void wait() {
    std::unique_lock<std::mutex> l(mu);
    const long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return gen != g; });
    }
  }
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Bar>> g_bars;
long g_next = 1;

// The collectives: every rank posts its send buffer, then reads the others'
// (sums in rank order); a second barrier keeps the buffers alive until all
// ranks have read them.
class EmuComm : public Comm {
 public:
  EmuComm(std::shared_ptr<Bar> b, int rank) : b_(b), rank_(rank) {}
  int barrier(cudaStream_t) override {
    b_->wait();
    return 0;
  }
  int reduce_scatter_v(const float* send, float* recv, const int64_t* b, cudaStream_t) override {
    b_->posted[rank_] = send;
    b_->wait();
    for (int64_t i = b[rank_]; i < b[rank_ + 1]; ++i) {
      float s = b_->posted[0][i];
      for (int q = 1; q < b_->world; ++q) s = s + b_->posted[q][i];
      recv[i - b[rank_]] = s;
    }
    b_->wait();
    return 0;
  }
  int all_gather_v(const float* send, float* recv, const int64_t* b, cudaStream_t) override {
    b_->posted[rank_] = send;
    b_->wait();
    for (int q = 0; q < b_->world; ++q)
      for (int64_t i = b[q]; i < b[q + 1]; ++i) recv[i] = b_->posted[q][i - b[q]];
    b_->wait();
    return 0;
  }
  int reduce_scatter(const float* send, float* recv, int64_t count, cudaStream_t) override {
    b_->posted[rank_] = send;
    b_->wait();
    for (int64_t i = 0; i < count; ++i) {
      const int64_t j = (int64_t)rank_ * count + i;
      float s = b_->posted[0][j];
      for (int q = 1; q < b_->world; ++q) s = s + b_->posted[q][j];
      recv[i] = s;
    }
    b_->wait();
    return 0;
  }
  int all_gather(const float* send, float* recv, int64_t count, cudaStream_t) override {
    b_->posted[rank_] = send;
    b_->wait();
    for (int q = 0; q < b_->world; ++q)
      for (int64_t i = 0; i < count; ++i) recv[(int64_t)q * count + i] = b_->posted[q][i];
    b_->wait();
    return 0;
  }
  std::string error() const override { return ""; }

 private:
  std::shared_ptr<Bar> b_;
  int rank_;
};

}  // namespace

int comm_unique_id(void* out, std::string*) {
  std::lock_guard<std::mutex> l(g_mu);
  memset(out, 0, kCommIdBytes);
  snprintf((char*)out, kCommIdBytes, "emu-%ld", g_next++);
  return 0;
}

Comm* comm_create(const void* id, int world, int rank, std::string*) {
  std::string key((const char*)id, strnlen((const char*)id, kCommIdBytes));
  std::lock_guard<std::mutex> l(g_mu);
  auto& b = g_bars[key];
  if (!b) {
    b = std::make_shared<Bar>();
    b->world = world;
    b->posted.assign(world, nullptr);
  }
  return new EmuComm(b, rank);
}

}  // namespace hp

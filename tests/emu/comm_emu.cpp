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

#include "../../paper_2005_14038_b200/csrc/comm.h"

namespace hp {
namespace {

struct Bar {
  std::mutex mu;
  std::condition_variable cv;
  int world = 0, arrived = 0;
  long gen = 0;
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

class EmuComm : public Comm {
 public:
  explicit EmuComm(std::shared_ptr<Bar> b) : b_(b) {}
  int barrier(cudaStream_t) override {
    b_->wait();
    return 0;
  }
  std::string error() const override { return ""; }

 private:
  std::shared_ptr<Bar> b_;
};

}  // namespace

int comm_unique_id(void* out, std::string*) {
  std::lock_guard<std::mutex> l(g_mu);
  memset(out, 0, kCommIdBytes);
  snprintf((char*)out, kCommIdBytes, "emu-%ld", g_next++);
  return 0;
}

Comm* comm_create(const void* id, int world, int, std::string*) {
  std::string key((const char*)id, strnlen((const char*)id, kCommIdBytes));
  std::lock_guard<std::mutex> l(g_mu);
  auto& b = g_bars[key];
  if (!b) {
    b = std::make_shared<Bar>();
    b->world = world;
  }
  return new EmuComm(b);
}

}  // namespace hp

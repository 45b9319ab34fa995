// capi.cpp -- extern "C" boundary of libhetpipe (include/hetpipe.h) and the
// deterministic tick controller (reading Z13).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/hetpipe.h"
#include "engine.h"

namespace hp {

// Tick controller: complete(p) = max(start(p) + lat_v, complete(p-1) + tau_v);
// the events of one tick run in the phases COMPLETE -> PUSH/APPLY -> GATE/PULL ->
// START, ascending VW inside a phase (reading Z5). A blocked VW is re-examined
// at every later tick ("may need to wait").
class Controller {
 public:
  explicit Controller(Engine* e) : e_(e) {}
  hp_status begin(const int64_t* tau, const int64_t* lat) {
    const auto& cfg = e_->cfg();
    const int N = cfg.num_vw;
    tau_.assign(tau, tau + N);
    lat_.resize(N);
    for (int v = 0; v < N; ++v) {
      if (tau_[v] < 1) return e_->fail(HP_ERR_INVALID, "tau must be >= 1");
      lat_[v] = lat ? lat[v] : (int64_t)cfg.Nm * tau_[v];
      if (lat_[v] < 1) return e_->fail(HP_ERR_INVALID, "lat must be >= 1");
    }
    // STARTs of a VW are scheduled in increasing p (ungated p+Nm after p's
    // COMPLETE, a gated START before its backlog, Z17), so only the latest
    // completion time per VW is needed -- never a table over all minibatches
    last_ct_.assign(N, -1);
    last_sp_.assign(N, 0);
    events_.clear();
    for (int v = 0; v < N; ++v)
      for (int64_t p = 1; p <= std::min<int64_t>(cfg.Nm, e_->last_p()); ++p) schedule(0, v, p);
    active_ = true;
    return HP_OK;
  }
  hp_status advance(int64_t target) {
    if (!active_) return e_->fail(HP_ERR_STATE, "hp_schedule_begin not called");
    while (!e_->done() && e_->commits() < target) {
      if (events_.empty()) return e_->fail(HP_ERR_STATE, "deadlock: no pending completion");
      if (hp_status st = tick()) return st;
    }
    // everything committed so far is launched; distributed contexts leave
    // their side streams running (the next advance's accumulation may overlap
    // this one's exchange): hp_flush / hp_sync join them to the context stream
    return e_->flush_queued();
  }
  void set_host_grads(const float* const* bufs, int n) { host_.assign(bufs, bufs + n); }
  bool host_grads() const { return !host_.empty(); }

 private:
  void schedule(int64_t t, int v, int64_t p) {
    // complete(p) = max(start(p) + L_v, complete(p-1) + tau_v) (Z13)
    int64_t ct = t + lat_[v];
    if (p > 1 && last_sp_[v] == p - 1) ct = std::max(ct, last_ct_[v] + tau_[v]);
    last_ct_[v] = ct;
    last_sp_[v] = p;
    events_[ct].push_back({v, p});
  }
  hp_status tick() {
    auto it = events_.begin();
    const int64_t t = it->first;
    std::vector<std::pair<int, int64_t>> comps = std::move(it->second);
    events_.erase(it);
    std::sort(comps.begin(), comps.end());
    e_->set_tick(t);
    const auto& cfg = e_->cfg();
    std::vector<std::pair<int, int64_t>> pushes;
    for (auto& vp : comps) {  // COMPLETE phase
      bool wave_end = false;
      const float* hg = nullptr;
      if (!host_.empty()) {
        const int64_t k = ((int64_t)vp.first * e_->last_p() + vp.second) % (int64_t)host_.size();
        hg = host_[k];
      }
      if (hp_status st = e_->complete(vp.first, vp.second, nullptr, hg, &wave_end)) return st;
      if (wave_end) pushes.push_back({vp.first, (vp.second - 1) / ((int64_t)cfg.Nm * cfg.update_freq)});
    }
    for (auto& vc : pushes)  // PUSH/APPLY phase
      if (hp_status st = e_->push(vc.first, vc.second)) return st;
    for (int v = 0; v < cfg.num_vw; ++v) {  // GATE/PULL phase
      if (!e_->at_gate(v)) continue;
      std::vector<int64_t> started;
      hp_status st = e_->admit(v, &started);
      if (st < 0) return st;
      for (int64_t p : started) schedule(t, v, p);
    }
    std::vector<std::pair<int, int64_t>> ungated;  // START phase
    if (hp_status st = e_->tick_end(&ungated)) return st;
    for (auto& vp : ungated) schedule(t, vp.first, vp.second);
    return HP_OK;
  }

  Engine* e_;
  std::vector<int64_t> tau_, lat_;
  std::vector<int64_t> last_ct_;   // per VW: completion time of its latest START
  std::vector<int64_t> last_sp_;   //   and that START's minibatch
  std::map<int64_t, std::vector<std::pair<int, int64_t>>> events_;
  std::vector<const float*> host_;
  bool active_ = false;
};

}  // namespace hp

struct hp_ctx {
  std::unique_ptr<hp::Engine> eng;
  std::unique_ptr<hp::Controller> ctl;
};

struct hp_graph {
  hp_ctx* ctx = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool launched = false;
  std::vector<void*> bufs;            // multi-tick descriptor buffers the graph reads
  cudaEvent_t done = nullptr;         // recorded after the launch
};

namespace {
std::string g_init_error;

hp_status guard_device(hp_ctx* ctx) {
  if (!ctx || !ctx->eng) return HP_ERR_INVALID;
  if (ctx->eng->sticky()) return ctx->eng->sticky();
  cudaSetDevice(ctx->eng->cfg().device);
  return HP_OK;
}
}  // namespace

#define HP_ENTRY(ctx)                              \
  if (hp_status _s = guard_device(ctx)) return _s; \
  try {
#define HP_EXIT(ctx)                                                  \
  }                                                                   \
  catch (const std::bad_alloc&) {                                     \
    return ctx->eng->fail(HP_ERR_OOM, "host allocation failed");      \
  }                                                                   \
  catch (...) {                                                       \
    return ctx->eng->fail(HP_ERR_INVALID, "unexpected C++ exception"); \
  }

extern "C" {

size_t hp_config_size(void) { return sizeof(hp_config); }

void hp_config_default(hp_config* c) {
  if (!c) return;
  memset(c, 0, sizeof *c);
  c->num_vw = 1;
  c->Nm = 1;
  c->D = 0;
  c->waves = 1 << 30;
  c->nparams = 0;
  c->param_begin = 0;
  c->param_count = -1;
  c->lr = 0.01f;
  c->momentum = 0.f;
  c->seed = 200514038ull;
  c->grad_mode = HP_GRAD_FLOAT;
  c->w0_mode = HP_W0_PHILOX;
  c->pull_policy = HP_PULL_EAGER;
  c->local_semantics = HP_LOCAL_STRICT;
  c->apply_mode = HP_APPLY_DEFERRED;
  c->acc_slots = 2;
  c->merge_ticks = 1;
  c->world = 1;
  c->rank = 0;
  c->vw_span = 1;
  c->device = 0;
  c->stream = nullptr;
  c->transport = HP_XPORT_PEER;
  c->update_freq = 1;
  c->conv_a = 0.5f;
  c->conv_sigma = 1.0f;
  c->reserved = 0;
  c->arena = nullptr;
}

}  // extern "C"

namespace {
const char* validate(hp_config& cfg) {
  if (cfg.param_count < 0) cfg.param_count = cfg.nparams - cfg.param_begin;
  const char* bad = nullptr;
  if (cfg.num_vw < 1 || cfg.num_vw > 8) bad = "num_vw must be 1..8";
  else if (cfg.Nm < 1 || cfg.Nm > 32) bad = "Nm must be 1..32";
  else if (cfg.D < 0) bad = "D must be >= 0";
  else if (cfg.waves < 1) bad = "waves must be >= 1";
  else if (cfg.nparams < 0 || cfg.nparams >= (1ll << 34)) bad = "nparams must be in [0, 2^34)";
  else if (cfg.param_begin < 0 || cfg.param_begin % 32) bad = "param_begin must be a multiple of 32";
  else if (cfg.param_count < 0 || cfg.param_begin + cfg.param_count > cfg.nparams) bad = "bad shard";
  else if (cfg.acc_slots < 2 || cfg.acc_slots > 8) bad = "acc_slots must be 2..8";
  else if (cfg.grad_mode < 0 || cfg.grad_mode > 3) bad = "bad grad_mode";

  else if (cfg.w0_mode < 0 || cfg.w0_mode > 1) bad = "bad w0_mode";
  else if (cfg.pull_policy < 0 || cfg.pull_policy > 1) bad = "bad pull_policy";
  else if (cfg.local_semantics < 0 || cfg.local_semantics > 1) bad = "bad local_semantics";
  else if (cfg.apply_mode < 0 || cfg.apply_mode > 1) bad = "bad apply_mode";
  else if (cfg.merge_ticks < 0 || cfg.merge_ticks > 1) bad = "bad merge_ticks";
  else if (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world) bad = "bad world/rank";
  else if (cfg.world > 8) bad = "world must be <= 8 (one NVLink domain of B200s)";
  else if (cfg.world > 1 && (cfg.vw_span < 1 || cfg.vw_span > cfg.world)) bad = "vw_span must be 1..world";
  else if (cfg.world > 1 && (cfg.param_begin != 0 || cfg.param_count != cfg.nparams))
    bad = "world > 1 places the whole model: param_begin 0, param_count -1";

  else if (cfg.transport < 0 || cfg.transport > 2) bad = "bad transport";
  else if (cfg.update_freq < 1 || cfg.update_freq > 64) bad = "update_freq must be 1..64";
  else if (cfg.lr_schedule < 0 || cfg.lr_schedule > 1) bad = "bad lr_schedule";
  else if (cfg.lr_schedule == HP_LR_THEOREM1 &&
           (int64_t)cfg.num_vw * cfg.waves * cfg.update_freq * cfg.Nm >= (1ll << 24))
    bad = "lr_schedule THEOREM1 needs num_vw * waves * F * Nm < 2^24 (t exact in fp32)";

  if (!bad && cfg.world > 1 && cfg.ps_bounds) {
    const int64_t* b = cfg.ps_bounds;
    if (b[0] != 0 || b[cfg.world] != cfg.nparams) bad = "ps_bounds must span [0, nparams]";
    for (int q = 1; q <= cfg.world && !bad; ++q)
      if (b[q] <= b[q - 1] || (q < cfg.world && b[q] % 32))
        bad = "ps_bounds must increase, inner bounds multiples of 32";
  }
  return bad;
}
}  // namespace

extern "C" {

int64_t hp_arena_bytes(const hp_config* cfg_in) {
  if (!cfg_in) return -1;
  hp_config cfg = *cfg_in;
  if (validate(cfg)) return -1;
  try {
    hp::Engine e(cfg);
    e.plan_layout();
    return e.arena_bytes();
  } catch (...) {
    return -1;
  }
}

hp_status hp_init_ex(hp_ctx** out, const hp_config* cfg_in) {
  if (!out || !cfg_in) return HP_ERR_INVALID;
  *out = nullptr;
  hp_config cfg = *cfg_in;
  const char* bad = validate(cfg);
  if (bad) {
    g_init_error = bad;
    return HP_ERR_INVALID;
  }
  hp_ctx* ctx = nullptr;
  try {
    ctx = new hp_ctx;
    ctx->eng.reset(new hp::Engine(cfg));
    ctx->ctl.reset(new hp::Controller(ctx->eng.get()));
  } catch (...) {
    delete ctx;
    g_init_error = "host allocation failed";
    return HP_ERR_OOM;
  }
  hp_status st = ctx->eng->init();
  if (st != HP_OK) {
    g_init_error = ctx->eng->error();
    delete ctx;
    return st;
  }
  *out = ctx;
  return HP_OK;
}

hp_status hp_init(hp_ctx** out, int32_t num_vw, int32_t Nm, int32_t D, int64_t nparams,
                  float lr) {
  hp_config c;
  hp_config_default(&c);
  c.num_vw = num_vw;
  c.Nm = Nm;
  c.D = D;
  c.nparams = nparams;
  c.lr = lr;
  return hp_init_ex(out, &c);
}

hp_status hp_accumulate_minibatch(hp_ctx* ctx, int32_t vw, int64_t p, const float* grad) {
  HP_ENTRY(ctx)
  return ctx->eng->complete(vw, p, grad, nullptr, nullptr);
  HP_EXIT(ctx)
}

hp_status hp_accumulate_minibatch_host(hp_ctx* ctx, int32_t vw, int64_t p,
                                       const float* host_grad) {
  HP_ENTRY(ctx)
  if (!host_grad) return ctx->eng->fail(HP_ERR_INVALID, "host_grad is NULL");
  return ctx->eng->complete(vw, p, nullptr, host_grad, nullptr);
  HP_EXIT(ctx)
}

hp_status hp_push_wave(hp_ctx* ctx, int32_t vw, int64_t c) {
  HP_ENTRY(ctx)
  return ctx->eng->push(vw, c);
  HP_EXIT(ctx)
}

hp_status hp_clock(hp_ctx* ctx, int32_t vw, int64_t* c_local, int64_t* c_global) {
  HP_ENTRY(ctx)
  return ctx->eng->clock(vw, c_local, c_global);
  HP_EXIT(ctx)
}

hp_status hp_pull(hp_ctx* ctx, int32_t vw) {
  HP_ENTRY(ctx)
  return ctx->eng->admit(vw, nullptr);
  HP_EXIT(ctx)
}

hp_status hp_tick_end(hp_ctx* ctx) {
  HP_ENTRY(ctx)
  return ctx->eng->tick_end(nullptr);
  HP_EXIT(ctx)
}

hp_status hp_flush(hp_ctx* ctx) {
  HP_ENTRY(ctx)
  return ctx->eng->flush_pending();
  HP_EXIT(ctx)
}

hp_status hp_comm_unique_id(void* out) {
  if (!out) return HP_ERR_INVALID;
  std::string err;
  if (hp::comm_unique_id(out, &err)) {
    g_init_error = err;
    return HP_ERR_COMM;
  }
  return HP_OK;
}

hp_status hp_ipc_handle(hp_ctx* ctx, void* out) {
  HP_ENTRY(ctx)
  if (!out) return ctx->eng->fail(HP_ERR_INVALID, "out is NULL");
  return ctx->eng->ipc_handle(out);
  HP_EXIT(ctx)
}

hp_status hp_connect(hp_ctx* ctx, const void* handles, const void* comm_id) {
  HP_ENTRY(ctx)
  if (!handles || !comm_id) return ctx->eng->fail(HP_ERR_INVALID, "NULL handles or id");
  return ctx->eng->connect(handles, comm_id);
  HP_EXIT(ctx)
}

hp_status hp_connect_symmetric(hp_ctx* ctx, const void* const* peer_bases, void* mc_base,
                               const void* comm_id) {
  HP_ENTRY(ctx)
  if (!peer_bases) return ctx->eng->fail(HP_ERR_INVALID, "NULL peer_bases");
  return ctx->eng->connect_symmetric(peer_bases, mc_base, comm_id);
  HP_EXIT(ctx)
}

hp_status hp_set_tick(hp_ctx* ctx, int64_t t) {
  HP_ENTRY(ctx)
  ctx->eng->set_tick(t);
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_schedule_begin(hp_ctx* ctx, const int64_t* tau, const int64_t* lat) {
  HP_ENTRY(ctx)
  if (!tau) return ctx->eng->fail(HP_ERR_INVALID, "tau is NULL");
  return ctx->ctl->begin(tau, lat);
  HP_EXIT(ctx)
}

hp_status hp_schedule_advance(hp_ctx* ctx, int64_t target, int64_t* commits) {
  HP_ENTRY(ctx)
  if (ctx->eng->graph_pending())
    return ctx->eng->fail(HP_ERR_STATE, "a captured graph has not been launched");
  hp_status st = ctx->ctl->advance(target);
  if (commits) *commits = ctx->eng->commits();
  return st;
  HP_EXIT(ctx)
}

hp_status hp_schedule_capture(hp_ctx* ctx, int64_t target, int64_t* commits, hp_graph** out) {
  HP_ENTRY(ctx)
  if (!out) return ctx->eng->fail(HP_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (ctx->ctl->host_grads()) return ctx->eng->fail(HP_ERR_STATE, "host gradients cannot be captured");
  if (hp_status st = ctx->eng->capture_begin()) return st;
  hp_status st = ctx->ctl->advance(target);
  cudaGraphExec_t exec = nullptr;
  if (hp_status st2 = ctx->eng->capture_end(st == HP_OK, &exec)) return st != HP_OK ? st : st2;
  if (commits) *commits = ctx->eng->commits();
  hp_graph* g = new hp_graph;
  g->ctx = ctx;
  g->exec = exec;
  g->bufs = ctx->eng->take_graph_bufs();
  *out = g;
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_graph_launch(hp_graph* g) {
  if (!g || !g->ctx) return HP_ERR_INVALID;
  hp_ctx* ctx = g->ctx;
  HP_ENTRY(ctx)
  if (g->launched) return ctx->eng->fail(HP_ERR_STATE, "graph already launched");
  g->launched = true;
  if (hp_status st = ctx->eng->graph_launch(g->exec)) return st;
  if (!g->bufs.empty()) {           // the buffers live until the graph has run
    cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming);
    cudaEventRecord(g->done, (cudaStream_t)ctx->eng->stream());
  }
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_launch_floor(hp_ctx* ctx, int32_t n, int32_t graph, float* us_per_launch) {
  HP_ENTRY(ctx)
  return ctx->eng->launch_floor(n, graph != 0, us_per_launch);
  HP_EXIT(ctx)
}

void hp_graph_destroy(hp_graph* g) {
  if (!g) return;
  if (g->done) {
    cudaEventSynchronize(g->done);
    cudaEventDestroy(g->done);
  }
  for (void* b : g->bufs) cudaFree(b);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
}

hp_status hp_run_schedule(hp_ctx* ctx, const int64_t* tau, const int64_t* lat) {
  HP_ENTRY(ctx)
  if (!tau) return ctx->eng->fail(HP_ERR_INVALID, "tau is NULL");
  if (hp_status st = ctx->ctl->begin(tau, lat)) return st;
  if (hp_status st = ctx->ctl->advance(INT64_MAX)) return st;
  return ctx->eng->flush_applies();
  HP_EXIT(ctx)
}

hp_status hp_schedule_set_host_grads(hp_ctx* ctx, const float* const* bufs, int32_t n) {
  HP_ENTRY(ctx)
  if (ctx->eng->cfg().grad_mode != HP_GRAD_EXTERNAL)
    return ctx->eng->fail(HP_ERR_STATE, "host gradients need HP_GRAD_EXTERNAL");
  if (!bufs || n < 1) return ctx->eng->fail(HP_ERR_INVALID, "no host buffers");
  for (int i = 0; i < n; ++i)
    if (!bufs[i]) return ctx->eng->fail(HP_ERR_INVALID, "NULL host buffer");
  ctx->ctl->set_host_grads(bufs, n);
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_drain(hp_ctx* ctx) {
  HP_ENTRY(ctx)
  return ctx->eng->drain();
  HP_EXIT(ctx)
}

hp_status hp_sync(hp_ctx* ctx) {
  HP_ENTRY(ctx)
  return ctx->eng->sync();
  HP_EXIT(ctx)
}

hp_status hp_read_weights(hp_ctx* ctx, int32_t which, int64_t offset, int64_t count,
                          float* host_dst) {
  HP_ENTRY(ctx)
  return ctx->eng->read(which, offset, count, host_dst);
  HP_EXIT(ctx)
}

hp_status hp_trace_dump(hp_ctx* ctx, const char* path) {
  HP_ENTRY(ctx)
  if (!path || !*path) return HP_OK;
  FILE* f = fopen(path, "w");
  if (!f) return ctx->eng->fail(HP_ERR_INVALID, "cannot open trace path");
  const std::string& t = ctx->eng->trace();
  size_t w = fwrite(t.data(), 1, t.size(), f);
  fclose(f);
  if (w != t.size()) return ctx->eng->fail(HP_ERR_INVALID, "short trace write");
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_trace_enable(hp_ctx* ctx, int32_t enable) {
  HP_ENTRY(ctx)
  ctx->eng->set_trace(enable != 0);
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_get_stats(hp_ctx* ctx, hp_stats* out) {
  HP_ENTRY(ctx)
  if (!out) return ctx->eng->fail(HP_ERR_INVALID, "out is NULL");
  ctx->eng->stats(out);
  return HP_OK;
  HP_EXIT(ctx)
}

hp_status hp_profile_enable(hp_ctx* ctx, int32_t enable) {
  HP_ENTRY(ctx)
  return ctx->eng->profile_enable(enable != 0);
  HP_EXIT(ctx)
}

hp_status hp_profile_read(hp_ctx* ctx, double* kernel_ms, double* alg_bytes, int64_t* launches) {
  HP_ENTRY(ctx)
  return ctx->eng->profile_read(kernel_ms, alg_bytes, launches);
  HP_EXIT(ctx)
}

hp_status hp_profile_launches(hp_ctx* ctx, int64_t max, float* ms, double* alg_bytes,
                              int32_t* shape, double* sync_bytes, float* start_ms,
                              int64_t* n) {
  HP_ENTRY(ctx)
  return ctx->eng->profile_launches(max, ms, alg_bytes, shape, sync_bytes, start_ms, n);
  HP_EXIT(ctx)
}

hp_status hp_profile_link(hp_ctx* ctx, int64_t max, double* link_bytes, int64_t* n) {
  HP_ENTRY(ctx)
  return ctx->eng->profile_link(max, link_bytes, n);
  HP_EXIT(ctx)
}

hp_status hp_profile_streams(hp_ctx* ctx, int64_t max, int32_t* stream_ids, int64_t* n) {
  HP_ENTRY(ctx)
  return ctx->eng->profile_streams(max, stream_ids, n);
  HP_EXIT(ctx)
}

hp_status hp_profile_sync_latency(hp_ctx* ctx, int64_t max, float* ms, int32_t* vw,
                                  int32_t* waited, int64_t* n) {
  HP_ENTRY(ctx)
  return ctx->eng->profile_sync(max, ms, vw, waited, n);
  HP_EXIT(ctx)
}

int64_t hp_s_global(int32_t Nm, int32_t D) {
  // s_global = (D+1)(s_local+1) + s_local - 1 with s_local = Nm-1
  return (int64_t)(D + 1) * Nm + (Nm - 1) - 1;
}

int64_t hp_s_global_f(int32_t Nm, int32_t D, int32_t F) {
  // F(D+1)(s_local+1) + (F-1)(s_local+1) + s_local - 1 = F(D+2)(s_local+1) - 2
  return (int64_t)F * (D + 2) * Nm - 2;
}

int64_t hp_version_floor(int64_t p, int32_t Nm, int32_t D) {
  const int64_t f = p - (hp_s_global(Nm, D) + 1);
  return f > 0 ? f : 0;
}

const char* hp_last_error(const hp_ctx* ctx) {
  if (!ctx || !ctx->eng) return g_init_error.c_str();
  return ctx->eng->error().c_str();
}

const char* hp_version(void) { return "hetpipe-wsp-b200 0.1 (sm_100a)"; }

void hp_finalize(hp_ctx* ctx) {
  if (!ctx) return;
  if (ctx->eng) cudaSetDevice(ctx->eng->cfg().device);
  delete ctx;
}

}  // extern "C"

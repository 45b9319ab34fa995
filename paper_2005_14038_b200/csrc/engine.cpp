// engine.cpp -- WSP protocol engine (see engine.h). Host C++; device work is
// one fused kernel launch per flushed batch (kernels.cu).
#include "engine.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

namespace hp {

namespace {
int64_t wave_of(int64_t p, int Nm) { return (p - 1) / Nm; }
}  // namespace

Engine::Engine(const hp_config& cfg) : cfg_(cfg) {
  N_ = cfg.num_vw;
  Nm_ = cfg.Nm;
  R_ = cfg.acc_slots;
  W_ = cfg.waves;
  U_ = (int64_t)Nm_ * cfg.update_freq;
  last_p_ = W_ * U_;
  begin_ = cfg.param_begin;
  n_ = cfg.param_count;
  vw_.resize(N_);
  G_ = cfg.world;
  rank_ = cfg.rank;
  span_ = cfg.vw_span;
  dist_ = G_ > 1;
  convex_ = cfg.grad_mode == HP_GRAD_CONVEX;
}

namespace {
// even contiguous split of [0, P) into n parts, inner boundaries multiples of 32
// floats, the last part takes the remainder (reading Z12)
std::vector<int64_t> even_bounds(int64_t P, int n) {
  const int64_t per = (P / n) / 32 * 32;
  std::vector<int64_t> b(n + 1);
  for (int i = 0; i < n; ++i) b[i] = per * i;
  b[n] = P;
  return b;
}
// ceil split: the first n-1 parts ceil(P/n) rounded up to 32 floats, the last
// the (smaller) rest -- equal blocks for NCCL's equal-count collectives
std::vector<int64_t> ceil_bounds(int64_t P, int n) {
  const int64_t per = ((P + n - 1) / n + 31) / 32 * 32;
  std::vector<int64_t> b(n + 1);
  for (int i = 0; i < n; ++i) b[i] = std::min<int64_t>(per * i, P);
  b[n] = P;
  return b;
}
size_t align256(int64_t nfloat) { return ((size_t)std::max<int64_t>(nfloat, 1) * 4 + 255) / 256 * 256; }
}  // namespace

// Placement (world G, span k): PS shard q = even_bounds(P, G)[q..q+1] on GPU q;
// VW v's stage j = even_bounds(P, k)[j..j+1] on GPU (v*k + j) mod G. k = G is the
// paper's ED-local placement (stage q = shard q); k = 1 a full
// replica per VW (one VW per GPU as in C5, or several).
RankLayout Engine::layout_of(int q) const {
  RankLayout L;
  L.s0 = shard_b_[q];
  L.s1 = shard_b_[q + 1];
  L.a.assign(N_, 0);
  L.len.assign(N_, 0);
  L.has.assign(N_, 0);
  L.wl_off.assign(N_, 0);
  L.acc_off.assign(N_, std::vector<size_t>(R_, 0));
  L.stash_off.assign(N_, std::vector<size_t>(cfg_.grad_mode == HP_GRAD_CONVEX ? Nm_ : 0, 0));
  L.snap_off.assign(N_, 0);
  // the shard regions are sized for the largest shard, so ranks holding
  // congruent VW sets have identical offsets (the multicast mapping of NVLS
  // addresses the same offset on every GPU)
  int64_t smax = 0;
  for (int r = 0; r < G_; ++r) smax = std::max(smax, shard_b_[r + 1] - shard_b_[r]);
  size_t off = 0;
  L.wg_off = off;
  off += align256(smax);
  if (cfg_.momentum != 0.f) {
    L.m_off = off;
    off += align256(smax);
  }
  if (cfg_.transport == HP_XPORT_NCCL && G_ > 1) {
    L.x_off = off;
    off += align256(smax);
  }
  for (int v = 0; v < N_; ++v) {
    for (int j = 0; j < span_; ++j) {
      if ((v * span_ + j) % G_ != q) continue;
      L.a[v] = stage_b_[j];
      L.len[v] = stage_b_[j + 1] - stage_b_[j];
      L.has[v] = 1;
      // NCCL transport with full replicas: w_local and the acc slots padded to
      // G x the largest shard, so ncclReduceScatter / ncclAllGather (equal
      // counts) work on them directly; the padding is never read back
      const int64_t alen = (cfg_.transport == HP_XPORT_NCCL && G_ > 1 && span_ == 1)
                               ? std::max<int64_t>(L.len[v], (int64_t)G_ * smax) : L.len[v];
      L.wl_off[v] = off;
      off += align256(alen);
      for (int r = 0; r < R_; ++r) {
        L.acc_off[v][r] = off;
        off += align256(alen);
      }
      for (auto& so : L.stash_off[v]) {
        so = off;
        off += align256(L.len[v]);
      }
      if (cfg_.update_freq > 1 && cfg_.local_semantics == HP_LOCAL_STRICT) {
        L.snap_off[v] = off;
        off += align256(L.len[v]);
      }
    }
  }
  if (G_ > 1) {                       // K7 flags: barrier, arrive, done; one uint64
    L.flag_off = off;                 // per source rank each
    off += align256(6 * G_);
  }
  L.bytes = off;
  return L;
}

Engine::~Engine() {
  delete comm_;
  for (void* b : graph_bufs_) cudaFree(b);
  if (up_) cudaStreamDestroy(up_);
  if (flag_err_) cudaFree(flag_err_);
  if (tiles_) cudaFree(tiles_);
  for (auto e : evpool_) cudaEventDestroy(e);
  if (xs_) cudaStreamDestroy(xs_);
  if (xs2_) cudaStreamDestroy(xs2_);
  for (auto v : vs_)
    if (v) cudaStreamDestroy(v);
  for (auto v : fs_)
    if (v) cudaStreamDestroy(v);
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  for (auto e : ev_) cudaEventDestroy(e);
  if (arena_ && !ext_arena_) cudaFree(arena_);
  for (auto& v : vw_)
    for (float* g : v.grad_ring) cudaFree(g);
  if (own_stream_ && stream_) cudaStreamDestroy(stream_);
}

hp_status Engine::fail(hp_status s, const std::string& msg) {
  err_ = msg;
  if (s == HP_ERR_CUDA) sticky_ = s;
  return s;
}

hp_status Engine::check_cuda(int err, const char* what) {
  if (err == cudaSuccess) return HP_OK;
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString((cudaError_t)err));
  return fail(HP_ERR_CUDA, buf);
}

void Engine::plan_layout() {
  if (dist_) {
    if (cfg_.ps_bounds) shard_b_.assign(cfg_.ps_bounds, cfg_.ps_bounds + G_ + 1);
    else if (cfg_.transport == HP_XPORT_NCCL && span_ == 1) shard_b_ = ceil_bounds(cfg_.nparams, G_);
    else shard_b_ = even_bounds(cfg_.nparams, G_);
    stage_b_ = even_bounds(cfg_.nparams, span_);
  } else {
    shard_b_ = {begin_, begin_ + n_};
    stage_b_ = {begin_, begin_ + n_};
    G_ = 1;
    span_ = 1;
    rank_ = 0;
  }
}

hp_status Engine::init() {
  if (cudaSetDevice(cfg_.device) != cudaSuccess) return check_cuda(cudaGetLastError(), "cudaSetDevice");
  if (hp_status st = check_cuda(preload_kernels(), "kernel preload")) return st;
  if (cfg_.stream) {
    stream_ = (cudaStream_t)cfg_.stream;
  } else {
    if (int e = cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking)) return check_cuda(e, "stream");
    own_stream_ = true;
  }
  {
    // small single-rank contexts run a capture's ticks through the multi-tick
    // kernel (HP_TICK_BATCH=0 disables; HP_TICK_BATCH_MAX_N: largest n)
    const char* tb = getenv("HP_TICK_BATCH");
    const char* tn = getenv("HP_TICK_BATCH_MAX_N");
    const int64_t max_n = tn ? atoll(tn) : (1 << 16);
    batch_ok_ = (!tb || atoi(tb) != 0) && cfg_.world <= 1 && cfg_.grad_mode != HP_GRAD_EXTERNAL &&
                cfg_.param_count > 0 && cfg_.param_count <= max_n;
  }
  if (const char* sv = getenv("HP_STRESS")) {
    const uint64_t seed = strtoull(sv, nullptr, 10);
    if (seed) stress_ = (seed * 0x9E3779B97F4A7C15ull) ^ (uint64_t)(cfg_.rank + 1) * 0xD1B54A32D192ED03ull;
    if (const char* us = getenv("HP_STRESS_US")) stress_ns_ = 1000ull * strtoull(us, nullptr, 10);
  }
  // arena: w_global, [m], per VW w_local + R acc slots; each 256-byte aligned.
  // Single-rank contexts own [param_begin, +param_count) of every buffer; with
  // world > 1 the placement layout decides (layout_of).
  plan_layout();
  cfg_.ps_bounds = nullptr;          // borrowed for hp_init_ex only (copied)
  for (int q = 0; q < G_; ++q) lay_.push_back(layout_of(q));
  const RankLayout& L = lay_[rank_];
  if (cfg_.arena) {
    if ((uintptr_t)cfg_.arena & 255) return fail(HP_ERR_INVALID, "arena not 256-byte aligned");
    arena_ = cfg_.arena;
    ext_arena_ = true;
  } else if (cudaMalloc(&arena_, L.bytes) != cudaSuccess) {
    cudaGetLastError();
    arena_ = nullptr;
    return fail(HP_ERR_OOM, "device arena allocation failed");
  }
  char* base = (char*)arena_;
  begin_ = L.s0;
  n_ = L.s1 - L.s0;
  wg_ = (float*)(base + L.wg_off);
  if (cfg_.momentum != 0.f) m_ = (float*)(base + L.m_off);
  for (int v = 0; v < N_; ++v) {
    VW& s = vw_[v];
    s.a0 = L.a[v];
    s.len = L.len[v];
    s.grad_of_slot.assign(Nm_, nullptr);
    s.here = L.has[v] != 0;
    if (!s.here) continue;
    s.wl = (float*)(base + L.wl_off[v]);
    for (int r = 0; r < R_; ++r) s.acc.push_back((float*)(base + L.acc_off[v][r]));
    for (size_t so : L.stash_off[v]) s.stash.push_back((float*)(base + so));
    if (L.snap_off[v]) s.snap = (float*)(base + L.snap_off[v]);
  }
  peer_.assign(G_, nullptr);
  peer_[rank_] = base;
  const uint32_t k0 = (uint32_t)(cfg_.seed & 0xffffffffu), k1 = (uint32_t)(cfg_.seed >> 32);
  hp_status st = check_cuda(
      launch_init(wg_, n_, begin_, cfg_.w0_mode, cfg_.grad_mode, k0, k1, stream_), "init");
  for (auto& v : vw_)
    if (st == HP_OK && v.here)
      st = check_cuda(launch_init(v.wl, v.len, v.a0, cfg_.w0_mode, cfg_.grad_mode, k0, k1, stream_),
                      "init");
  if (st == HP_OK && m_) st = check_cuda(cudaMemsetAsync(m_, 0, (size_t)n_ * 4, stream_), "memset");
  if (st == HP_OK) {
    if (cudaMalloc((void**)&tiles_, kTileSlots * 128) != cudaSuccess) {
      cudaGetLastError();
      tiles_ = nullptr;
      return fail(HP_ERR_OOM, "tile counter allocation failed");
    }
    st = check_cuda(cudaMemsetAsync(tiles_, 0, kTileSlots * 128, stream_), "tile counters");
  }
  if (st == HP_OK && G_ > 1)            // K7 flags start at epoch 0 (before hp_connect's barrier)
    st = check_cuda(cudaMemsetAsync(base + L.flag_off, 0, (size_t)G_ * 24, stream_), "flags");
  for (auto& v : vw_)                 // CONVEX: minibatches 1..Nm read w0
    for (float* sl : v.stash)
      if (st == HP_OK)
        st = check_cuda(cudaMemcpyAsync(sl, v.wl, (size_t)v.len * 4, cudaMemcpyDeviceToDevice,
                                        stream_), "stash init");
  if (st != HP_OK) return st;
  // minibatches 1..Nm of every VW start at t=0 with w0
  for (int v = 0; v < N_; ++v) {
    for (int64_t p = 1; p <= std::min<int64_t>(Nm_, last_p_); ++p) {
      vw_[v].started = p;
      rec('S', v, "START", p, wave_of(p, U_));
    }
  }
  return check_cuda(cudaStreamSynchronize(stream_), "init sync");
}

void Engine::rec(char phase, int v, const char* kind, int64_t p, int64_t c) {
  if (!trace_on_) return;
  const VW& s = vw_[v];
  char buf[192];
  int n = snprintf(buf, sizeof buf, "%lld %c %d %s %lld %lld %lld %lld %lld %lld %lld\n",
                   (long long)tick_, phase, v, kind, (long long)p, (long long)c,
                   (long long)s.c_local, (long long)c_global_, (long long)s.a,
                   (long long)s.held_g, (long long)s.held_K);
  trace_.append(buf, n);
}

std::pair<bool, bool> Engine::gate_open(int v) const {
  const VW& s = vw_[v];
  const bool within = s.c_local - c_global_ <= cfg_.D;
  if (cfg_.pull_policy == HP_PULL_EAGER) return {within, true};
  if (s.held_g >= s.c_local - cfg_.D) return {true, false}; // held version suffices
  return {within, true};
}

bool Engine::done() const {
  for (const auto& s : vw_)
    if (s.c_local < W_) return false;
  return true;
}

void Engine::fill_fold(DFold& f, int v, int64_t x) const {
  const int64_t q = x > 0 ? x : -x;
  f.v = (uint32_t)v;
  f.p = (uint32_t)q;
  f.op = x > 0 ? 0u : 1u;
  f.grad = x > 0 ? fold_grad(v, q) : nullptr;
  f.neg_lr = neg_lr_of(v, q);
  f.stash = convex_ ? vw_[v].stash[(q - 1) % Nm_] : nullptr;
}

float Engine::neg_lr_of(int v, int64_t p) const {
  if (cfg_.lr_schedule == HP_LR_CONSTANT) return -cfg_.lr;
  // eta_t = sigma / sqrt(t) (Theorem 1): fl(sqrt) and
  // fl(/) are correctly rounded IEEE ops, t < 2^24 is exact in fp32; negation
  // is exact
  const float t = (float)((p - 1) * (int64_t)N_ + v + 1);
  return -(cfg_.lr / sqrtf(t));
}

const float* Engine::fold_grad(int v, int64_t p) const {
  if (cfg_.grad_mode != HP_GRAD_EXTERNAL) return nullptr;
  return vw_[v].grad_of_slot[(p - 1) % Nm_];
}

// ---------------------------------------------------------------------------
hp_status Engine::complete(int v, int64_t p, const float* grad_dev, const float* grad_host,
                           bool* wave_end_out) {
  if (sticky_) return sticky_;
  if (v < 0 || v >= N_) return fail(HP_ERR_INVALID, "vw out of range");
  if (dist_ && !connected_) return fail(HP_ERR_STATE, "distributed context not connected (hp_connect)");
  VW& s = vw_[v];
  if (p != s.completed + 1 || p > s.started || p > last_p_)
    return fail(HP_ERR_PROTOCOL, "COMPLETE out of order or minibatch not started");
  const bool ext = cfg_.grad_mode == HP_GRAD_EXTERNAL;
  if (ext && !grad_dev && !grad_host) return fail(HP_ERR_INVALID, "EXTERNAL mode needs a gradient");
  if (!ext && (grad_dev || grad_host)) return fail(HP_ERR_INVALID, "gradient given in synthetic mode");
  if (grad_dev && ((uintptr_t)grad_dev & 15)) return fail(HP_ERR_INVALID, "gradient not 16-byte aligned");
  // phase order inside a batch: COMPLETE < PUSH < PULL; one COMPLETE per VW;
  // CONVEX: a complete reads w_p from its stash slot in phase B, so a pending
  // STASH of this VW (phase D) must be on the device first
  bool again = phase_ > kPhComplete;
  for (auto& b : bc_) again |= b.v == v;
  if (convex_)
    for (int64_t q : s.pending_folds) again |= q < 0;
  if ((int)bc_.size() >= kMaxC && !again) desc_splits_++;
  if (again || (int)bc_.size() >= kMaxC)
    if (hp_status st = flush()) return st;
  const int64_t c = wave_of(p, U_);            // the clock p belongs to (F waves)
  const int slot = (int)(c % R_);
  const bool first = (p - 1) % U_ == 0;
  // F > 1, STRICT: the first completion joining a waiting VW's open clock
  // snapshots that clock's aggregate for the pull (reading Z25): its launch
  // copies the acc it loads, before adding u (kSnapAcc)
  const bool snap = s.at_gate && U_ > Nm_ && cfg_.local_semantics == HP_LOCAL_STRICT &&
                    s.backlog.empty() && s.acc_count > 0 && !first;
  if (snap) s.snap_valid = true;
  if (first) {  // the slot must not hold a pushed wave that is not applied yet
    bool busy = false;
    for (auto& a : pending_applies_) busy |= (a.v == v && a.slot == slot);
    for (auto& a : ba_) busy |= (a.v == v && a.slot == slot);
    if (busy) {
      if (hp_status st = flush()) return st;
      if (hp_status st = flush_applies()) return st;
    }
  }
  const float* g = grad_dev;
  if (grad_host && dist_ && !s.here) {   // the VW has no stage on this rank
    grad_host = nullptr;
    g = nullptr;
  }
  if (grad_host && capturing_) return fail(HP_ERR_STATE, "host gradients cannot be captured");
  if (grad_host) {  // library-owned device copy of a host gradient
    if (s.grad_ring.empty()) {
      s.grad_ring.assign(Nm_, nullptr);
    }
    float*& dst = s.grad_ring[(p - 1) % Nm_];
    if (!dst && cudaMalloc(&dst, (size_t)std::max<int64_t>(s.len, 1) * 4) != cudaSuccess) {
      cudaGetLastError();
      dst = nullptr;
      return fail(HP_ERR_OOM, "gradient staging allocation failed");
    }
    // a distributed placement's host gradient is the VW's whole model: copy
    // this rank's stage of it (single-rank contexts: their shard, a0 = begin).
    // Distributed: the copy runs on the VW's accumulation stream (the complete
    // that reads it follows in stream order) after every exchange-stream and
    // fold-stream op issued so far (a deferred fold may still read the slot)
    const float* src = dist_ ? grad_host + s.a0 : grad_host;
    // the slot's previous minibatch (p - Nm) may still have its fold queued on
    // the host (e.g. replayed at an admission in this batch): launch it first,
    // it reads the gradient this copy replaces
    bool reader_queued = false;
    for (int64_t x : s.pending_folds) reader_queued |= x > 0 && (x - 1) % Nm_ == (p - 1) % Nm_;
    if (reader_queued)
      if (hp_status st = flush()) return st;
    cudaStream_t cst = stream_;
    if (dist_) {
      fork_streams();
      cst = vs_[v];
      for (cudaStream_t o : {xs_, fs_[v]}) {
        if (!o) continue;                 // no fold stream (HP_SPLIT_FOLDS off)
        cudaEvent_t e = pool_event();
        cudaEventRecord(e, o);
        cudaStreamWaitEvent(cst, e, 0);
      }
    }
    stress(cst);
    if (hp_status st = check_cuda(cudaMemcpyAsync(dst, src, (size_t)s.len * 4,
                                                  cudaMemcpyHostToDevice, cst), "H2D grad"))
      return st;
    g = dst;
  }
  if (ext) s.grad_of_slot[(p - 1) % Nm_] = g;
  phase_ = kPhComplete;
  const bool wave_end = p % U_ == 0;          // the clock's last minibatch: push
  // START(p+Nm) is the gated one iff p+Nm = (c+2)*U (with F)
  const bool gated_next = (p + Nm_) % U_ == 0 && p + Nm_ >= 2 * U_ && p + Nm_ <= last_p_;
  bc_.push_back({v, p, slot, first, wave_end, g, snap});
  s.completed = p;
  s.acc_count = first ? 1 : s.acc_count + 1;
  if (!s.at_gate) {
    s.pending_folds.push_back(p);          // w_local = w_local + u_p
    s.a = p;
    if (gated_next) {                      // evaluated in this tick's GATE phase
      s.at_gate = true;
      s.snap_valid = false;
    } else if (p + Nm_ <= last_p_) {       // START(p+Nm) without waiting
      s.started = p + Nm_;
      ungated_.push_back({v, p + Nm_});
      if (convex_) s.pending_folds.push_back(-(p + Nm_));
    }
  } else {                                  // waiting at the gate (Z17)
    s.backlog.push_back(p);
    if (cfg_.local_semantics == HP_LOCAL_AT_LEAST) {
      s.pending_folds.push_back(p);
      s.a = p;
    }
  }
  rec('C', v, "COMPLETE", p, c);
  if (wave_end_out) *wave_end_out = wave_end;
  return HP_OK;
}

hp_status Engine::push(int v, int64_t c) {
  if (sticky_) return sticky_;
  if (v < 0 || v >= N_) return fail(HP_ERR_INVALID, "vw out of range");
  VW& s = vw_[v];
  if (c != s.c_local) return fail(HP_ERR_PROTOCOL, "duplicate or out-of-order push");
  if (s.completed < (c + 1) * U_) return fail(HP_ERR_PROTOCOL, "push of an incomplete wave");
  if (phase_ > kPhPush)
    if (hp_status st = flush()) return st;
  phase_ = kPhPush;
  commit_.push_back({v, c});
  pending_applies_.push_back({v, c, (int)(c % R_)});
  s.c_local = c + 1;
  int64_t mn = vw_[0].c_local;
  for (auto& x : vw_) mn = std::min(mn, x.c_local);
  c_global_ = mn;
  s.acc_count = 0;
  if (cfg_.apply_mode == HP_APPLY_ON_ARRIVAL) {        // apply on receipt
    for (auto& a : pending_applies_) ba_.push_back(a);
    pending_applies_.clear();
  }
  rec('P', v, "PUSH", (c + 1) * U_, c);
  return HP_OK;
}

hp_status Engine::clock(int v, int64_t* cl, int64_t* cg) {
  if (sticky_) return sticky_;
  if (v < 0 || v >= N_) return fail(HP_ERR_INVALID, "vw out of range");
  if (cl) *cl = vw_[v].c_local;
  if (cg) *cg = c_global_;
  if (vw_[v].at_gate && !gate_open(v).first) return HP_WOULD_BLOCK;
  return HP_OK;
}

hp_status Engine::admit(int v, std::vector<int64_t>* started) {
  if (sticky_) return sticky_;
  if (v < 0 || v >= N_) return fail(HP_ERR_INVALID, "vw out of range");
  VW& s = vw_[v];
  if (!s.at_gate) return fail(HP_ERR_PROTOCOL, "pull outside the gate");
  const auto open = gate_open(v);
  const int64_t c = s.c_local - 1;
  const int64_t gated_p = (s.c_local + 1) * U_;      // (c+2)*U
  if (!open.first) {
    if (!s.blocked) {
      s.blocked = true;
      s.t_block = tick_;
      rec('G', v, "BLOCK", gated_p, c);
    }
    return HP_WOULD_BLOCK;
  }
  phase_ = kPhPull;
  s.waited_last = s.blocked;
  if (s.blocked) {
    s.wait += tick_ - s.t_block;
    s.blocked = false;
  }
  // CONVEX: a START recorded before this pull must read the pre-pull w_local
  // (never the case in the tick model: STARTs wait while the VW is at its
  // gate; kept as a guard)
  if (open.second && convex_) {
    bool stash_due = false;
    for (int64_t q : s.pending_folds) stash_due |= q < 0;
    if (stash_due)
      if (hp_status st = flush()) return st;
  }
  s.at_gate = false;
  if (open.second) {                                  // PULL
    for (auto& a : pending_applies_) ba_.push_back(a); // w_global must be current
    pending_applies_.clear();
    bpull_.push_back(v);
    auto& pf = s.pending_folds;
    s.pull_partial = nullptr;
    if (cfg_.local_semantics == HP_LOCAL_STRICT) {
      // own updates up to gated_p - Nm: the pushed ones are in w_global, those
      // of the open clock (F > 1 only) come as their aggregate (reading Z25);
      // folds they cover die
      const int64_t pushed_to = s.c_local * U_, gate_a = gated_p - Nm_;
      pf.erase(std::remove_if(pf.begin(), pf.end(),
                              [&](int64_t q) { return q > 0 && q <= gate_a; }),
               pf.end());
      if (gate_a > pushed_to && s.here)
        s.pull_partial = s.snap_valid ? s.snap : s.acc[s.c_local % R_];
      s.a = gate_a;
    } else {
      pf.clear();                                     // in w_global or the partial u~
      if (s.acc_count > 0 && s.here) s.pull_partial = s.acc[s.c_local % R_];
      s.a = s.completed;
    }
    s.snap_valid = false;
    s.held_g = c_global_;
    s.held_K = (int64_t)commit_.size();
    s.pulls++;
    rec('G', v, "PULL", gated_p, c);
  } else {
    rec('G', v, "ADMIT", gated_p, c);
  }
  s.started = gated_p;
  rec('G', v, "START", gated_p, wave_of(gated_p, U_));
  if (convex_) s.pending_folds.push_back(-gated_p);
  if (started) started->push_back(gated_p);
  for (int64_t q : s.backlog) {                       // Z17: replay in order
    if (cfg_.local_semantics == HP_LOCAL_STRICT) {
      s.pending_folds.push_back(q);
      s.a = q;
      rec('G', v, "FOLD", q, wave_of(q, U_));
    }
    if (q + Nm_ <= last_p_) {
      s.started = q + Nm_;
      rec('G', v, "START", q + Nm_, wave_of(q + Nm_, U_));
      if (convex_) s.pending_folds.push_back(-(q + Nm_));
      if (started) started->push_back(q + Nm_);
    }
  }
  s.backlog.clear();
  return HP_OK;
}

hp_status Engine::tick_end(std::vector<std::pair<int, int64_t>>* ungated) {
  if (sticky_) return sticky_;
  for (auto& vp : ungated_) {
    rec('S', vp.first, "START", vp.second, wave_of(vp.second, U_));
    if (ungated) ungated->push_back(vp);
  }
  ungated_.clear();
  ticks++;
  // Independent ops of consecutive ticks (disjoint VW state) may share a launch:
  // the batch is flushed by the first op that would conflict (complete.. checks)
  // or by the controller before it returns, so every buffer still passes through
  // exactly the states of the tick model.
  return cfg_.merge_ticks ? HP_OK : flush();
}

// ---------------------------------------------------------------------------
// Batch -> TickDesc(s). Algorithmic bytes are counted from the descriptor: each
// buffer read or written once per launch = 4 bytes per param of the launch's
// range [begin, begin+n); reads through peer segments are also NVLink bytes.
hp_status Engine::emit(TickDesc& d, int64_t begin, int64_t n, cudaStream_t st, int max_blocks,
                       double link_bytes) {
  if (!st) st = stream_;
  d.n = n;
  d.blk_base = begin >> 2;
  // an apply launch over a sub-range of this rank's shard addresses w_global
  // (and m) from the sub-range's start
  const int64_t woff = (d.na > 0 && begin > begin_ && begin < begin_ + n_) ? begin - begin_ : 0;
  d.wg = wg_ + woff;
  d.m = m_ ? m_ + woff : nullptr;
  d.neg_lr = -cfg_.lr;
  d.mu = cfg_.momentum;
  d.conv_a = cfg_.conv_a;
  d.conv_sigma = cfg_.conv_sigma;
  d.key0 = (uint32_t)(cfg_.seed & 0xffffffffu);
  d.key1 = (uint32_t)(cfg_.seed >> 32);
  bool any_pull = false, apply_now = false;
  for (int g = 0; g < d.ng; ++g) any_pull |= d.g[g].pull == 1;
  for (int j = 0; j < d.nc; ++j) apply_now |= (d.c[j].flags & kApplyNow) != 0;
  d.wg_store = (d.na > 0 || apply_now) ? 1 : 0;
  d.wg_load = (d.wg_store || any_pull) ? 1 : 0;
  if (d.nc == 0 && d.na == 0 && d.ng == 0) return HP_OK;
  const int streams = tick_streams(d);
  double pstore = 0, rstore = 0;         // owner-side pull stores (all / to peers)
  for (int k = 0; k < d.np; ++k) {
    pstore += 4.0 * (double)(d.pd[k].hi - d.pd[k].lo);
    const char* p0 = (const char*)(d.pd[k].ptr + d.pd[k].lo);
    const char* alo = (const char*)arena_;
    if (p0 < alo || p0 >= alo + lay_[rank_].bytes) rstore += 4.0 * (double)(d.pd[k].hi - d.pd[k].lo);
  }
  const double bytes = 4.0 * (double)n * streams + pstore;
  // remote (NVLink) reads: segments whose pointer is outside this rank's arena
  double remote = 0;
  const char* lo = (const char*)arena_;
  const char* hi = lo + lay_[rank_].bytes;
  for (int k = 0; k < d.na; ++k)
    for (int t = d.a[k].seg_begin; t < d.a[k].seg_end; ++t) {
      const int64_t b = t == d.a[k].seg_begin ? 0 : d.s[t - 1].end;
      const char* p = (const char*)(d.s[t].ptr + b);
      if (p < lo || p >= hi) remote += 4.0 * (double)(d.s[t].end - b);
    }
  for (int t = d.wgs_begin; t < d.wgs_end && d.wg_load; ++t) {
    const int64_t b = t == d.wgs_begin ? 0 : d.s[t - 1].end;
    const char* p = (const char*)(d.s[t].ptr + b);
    if (p < lo || p >= hi) remote += 4.0 * (double)(d.s[t].end - b);
  }
  for (int g = 0; g < d.ng; ++g)
    if (d.g[g].pull == 2)
      for (int t = d.g[g].seg_begin; t < d.g[g].seg_end; ++t) {
        const int64_t b = t == d.g[g].seg_begin ? 0 : d.s[t - 1].end;
        const char* p = (const char*)(d.s[t].ptr + b);
        if (p < lo || p >= hi) remote += 4.0 * (double)(d.s[t].end - b);
      }
  // L2 prefetch one chunk round ahead (HP_PREFETCH = distance in rounds, 0 off):
  // only for launches whose loads are all local (a hint; never a peer address)
  // and that have at most HP_PREFETCH_MAXLOADS load streams per chunk. Measured
  // on B200 (profiles/r01_prefetch_ab.txt): +3-7% on C2's 1-3 stream launches,
  // -1 to -7% on 4-6 stream ones, whose own loads already fill the memory system.
  static const int pf_env = getenv("HP_PREFETCH") ? atoi(getenv("HP_PREFETCH")) : 1;
  static const int pf_max = getenv("HP_PREFETCH_MAXLOADS") ? atoi(getenv("HP_PREFETCH_MAXLOADS")) : 3;
  int loads = d.wg_load + ((d.m && d.wg_store) ? 1 : 0) + d.na;
  for (int j = 0; j < d.nc; ++j)
    loads += ((d.c[j].flags & kLoadAcc) ? 1 : 0) + ((d.c[j].flags & kFoldInline) ? 1 : 0) +
             (d.c[j].grad ? 1 : 0) + (d.c[j].stash ? 1 : 0);
  for (int g = 0; g < d.ng; ++g) {
    loads += (d.g[g].pull != 1 ? 1 : 0) + ((d.g[g].pull && d.g[g].partial) ? 1 : 0);
    for (int k = d.g[g].f_begin; k < d.g[g].f_end; ++k)
      loads += (d.f[k].grad ? 1 : 0) + ((d.f[k].stash && d.f[k].op != 1) ? 1 : 0);
  }
  d.pf = (remote == 0 && loads <= pf_max) ? pf_env : 0;
  // (completes-only launches take the lean instance, set below with the tiles)
  // dynamic tile scheduling (HP_DYN, default on) for launches with at least
  // HP_DYN_MINLOADS load streams (HP_DYN_PULLS: also launches with pull groups):
  // counters of this launch stream
  static const int dyn_env = getenv("HP_DYN") ? atoi(getenv("HP_DYN")) : 1;
  static const int dyn_min = getenv("HP_DYN_MINLOADS") ? atoi(getenv("HP_DYN_MINLOADS")) : 2;
  static const int dyn_pulls = getenv("HP_DYN_PULLS") ? atoi(getenv("HP_DYN_PULLS")) : 1;
  // (small launches take the static grid: a tile claim is a chain of L2
  // atomics that costs more than a 4096-param tick, C1)
  static const int64_t dyn_n = getenv("HP_DYN_MIN_N") ? atoll(getenv("HP_DYN_MIN_N")) : (1 << 20);
  d.ctr = nullptr;
  d.done = nullptr;
  // completes-only launches take the lean instance, with dynamic tiles
  // whatever their load streams (HP_LEAN_DYN, default on: the 1-stream
  // complete otherwise runs a static grid and ends with its slowest CTA; C3 at
  // 4 GPUs 1.091 -> 1.074 ms, C2 neutral, profiles/r02/lean_dyn_ab/)
  static const int lean_env = getenv("HP_LEAN") ? atoi(getenv("HP_LEAN")) : 1;
  static const int lean_dyn = getenv("HP_LEAN_DYN") ? atoi(getenv("HP_LEAN_DYN")) : 1;
  d.lean = (lean_env && d.nc > 0 && d.na == 0 && d.ng == 0 && d.np == 0 && !d.wg_load &&
            !d.wg_store) ? 1 : 0;
  if (dyn_env && (loads >= dyn_min || (d.lean && lean_dyn)) && n >= dyn_n &&
      (dyn_pulls || d.ng == 0))
    tile_slot(st, &d.ctr, &d.done);
  if (capturing_ && batch_ok_ && st == stream_) {
    batch_.push_back(TickDescPad{d});
    alg_bytes_ += bytes;
    if (batch_.size() >= kTickBatch) return flush_batch();
    return HP_OK;
  }
  stress(st);
  prof_begin(st);
  int err = launch_tick(d, cfg_.grad_mode, m_ != nullptr, st, max_blocks);
  int inl = 0;
  for (int j = 0; j < d.nc; ++j) inl += (d.c[j].flags & kFoldInline) ? 1 : 0;
  int pulls = 0;
  for (int g = 0; g < d.ng; ++g) pulls |= d.g[g].pull != 0;
  prof_end(st, bytes, 4.0 * (double)n * tick_sync_streams(d) + pstore,
           d.nc | (inl << 4) | (d.na << 8) | (d.ng << 16) | (d.nf << 24) |
               (int)((unsigned)pulls << 31),
           link_bytes >= 0 ? link_bytes : std::max(remote, rstore));
  note_sync(d);
  launches_++;
  alg_bytes_ += bytes;
  nvl_bytes_ += remote;
  return check_cuda(err, "tick kernel");
}

bool Engine::tile_slot(cudaStream_t st, unsigned long long** ctr, unsigned int** done) {
  size_t i = 0;
  while (i < tile_streams_.size() && tile_streams_[i] != st) ++i;
  if (i == tile_streams_.size()) {
    if (!tiles_ || i >= (size_t)kTileSlots) return false;   // static grid stride instead
    tile_streams_.push_back(st);
  }
  *ctr = (unsigned long long*)(tiles_ + 128 * i);
  *done = (unsigned int*)(tiles_ + 128 * i + 64);
  return true;
}

// Wave-sync latency bookkeeping (profile window only): a launch with VW v's
// wave-end COMPLETE starts v's push; the launch that writes v's pulled
// w_local ends its sync (SURVEY.md 8(d) "wave-sync latency").
void Engine::note_sync(const TickDesc& d) {
  if (!prof_on_ || prof_launches_ == 0) return;
  const int64_t idx = prof_launches_ - 1;
  for (int j = 0; j < d.nc; ++j)
    if (d.c[j].flags != kFoldInline &&          // (a fold-only complete pushes nothing)
        d.c[j].p % (uint32_t)U_ == 0 && push_launch_[d.c[j].v] < 0)
      push_launch_[d.c[j].v] = idx;
  std::vector<int> pulled;
  for (int g = 0; g < d.ng; ++g)
    if (d.g[g].pull)
      for (int v = 0; v < N_; ++v)
        if (vw_[v].wl == d.g[g].wl) pulled.push_back(v);
  note_pulls(pulled);
}

void Engine::note_pulls(const std::vector<int>& vws) {
  if (!prof_on_ || prof_launches_ == 0) return;
  const int64_t idx = prof_launches_ - 1;
  for (int v : vws)
    if (push_launch_[v] >= 0) {
      sync_recs_.push_back({v, push_launch_[v], idx, vw_[v].waited_last ? 1 : 0});
      push_launch_[v] = -1;
    }
}

hp_status Engine::profile_sync(int64_t max, float* ms, int32_t* vw, int32_t* waited,
                               int64_t* n) {
  if (sticky_) return sticky_;
  if (hp_status st = join_exchange()) return st;
  if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "profile sync")) return st;
  const int64_t cnt = std::min<int64_t>(max, (int64_t)sync_recs_.size());
  for (int64_t i = 0; i < cnt; ++i) {
    float t = 0;
    const SyncRec& r = sync_recs_[i];
    if (int e = cudaEventElapsedTime(&t, ev_[2 * r.from], ev_[2 * r.to + 1])) return check_cuda(e, "elapsed");
    if (ms) ms[i] = t;
    if (vw) vw[i] = r.v;
    if (waited) waited[i] = r.waited;
  }
  if (n) *n = cnt;
  return HP_OK;
}

// The stream-ordered barrier of the exchange stream, profiled like a launch
// (shape nf = 126) so its cost shows in the launch mix.
// The stream-ordered barrier of the exchange stream:
// every rank stores the barrier's epoch into its slot of every peer's flag
// array (NVLink stores, release) and waits until its own array holds the
// epoch from every rank (acquire) -- one tiny kernel, no NCCL call. A wait
// that exceeds its deadline sets a device error flag, reported as
// HP_ERR_COMM at the next synchronising call. HP_FLAG_BARRIER=0 uses a
// 4-byte NCCL all-reduce instead. Profiled like a launch (shape nf = 126).
void Engine::stress(cudaStream_t st) {
  if (!stress_) return;
  stress_ ^= stress_ << 13;
  stress_ ^= stress_ >> 7;
  stress_ ^= stress_ << 17;
  if (stress_ & 1) return;
  launch_spin((stress_ >> 8) % (stress_ns_ + 1), st);
}

hp_status Engine::xbarrier() {
  stress(xs_);
  prof_begin(xs_);
  if (flag_barrier_) {
    ++epoch_;
    FlagBarrier fb;
    memset(&fb, 0, sizeof fb);
    fb.G = G_;
    fb.me = rank_;
    fb.epoch = epoch_;
    fb.err = flag_err_;
    fb.timeout_ns = flag_timeout_ns_;
    for (int q = 0; q < G_; ++q)
      fb.flags[q] = (unsigned long long*)(peer_[q] + lay_[q].flag_off);
    if (int e = launch_flag_barrier(fb, xs_)) return check_cuda(e, "flag barrier");
  } else if (!comm_ || comm_->barrier(xs_) != 0) {
    return fail(HP_ERR_COMM, comm_ ? comm_->error() : "no communicator for the NCCL barrier");
  }
  prof_end(xs_, 0.0, 0.0, 126 << 24);
  return HP_OK;
}

// Per-launch CUDA events of the profile window (hp_profile_enable).
void Engine::prof_begin(cudaStream_t st) {
  if (!prof_on_) return;
  while (ev_.size() < ev_used_ + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    ev_.push_back(e);
  }
  cudaEventRecord(ev_[ev_used_], st);
}

void Engine::prof_end(cudaStream_t st, double bytes, double sync_bytes, int32_t shape,
                      double link_bytes) {
  if (!prof_on_ || ev_.size() < ev_used_ + 2) return;
  cudaEventRecord(ev_[ev_used_ + 1], st);
  ev_used_ += 2;
  prof_bytes_ += bytes;
  prof_launches_++;
  prof_launch_bytes_.push_back(bytes);
  prof_launch_sync_.push_back(sync_bytes);
  prof_launch_shape_.push_back(shape);
  prof_launch_link_.push_back(link_bytes);
  prof_launch_stream_.push_back(stream_id(st));
}

int32_t Engine::stream_id(cudaStream_t st) const {
  if (st == stream_) return 0;
  if (st == xs_) return 1;
  if (st == xs2_) return 2;
  for (int v = 0; v < (int)vs_.size(); ++v) {
    if (st == vs_[v]) return 3 + v;
    if (fs_[v] && st == fs_[v]) return 3 + N_ + v;
  }
  return -1;
}

hp_status Engine::profile_streams(int64_t max, int32_t* ids, int64_t* n) {
  if (sticky_) return sticky_;
  const int64_t cnt = std::min<int64_t>(max, (int64_t)prof_launch_stream_.size());
  for (int64_t i = 0; i < cnt && ids; ++i) ids[i] = prof_launch_stream_[i];
  if (n) *n = cnt;
  return HP_OK;
}

hp_status Engine::profile_link(int64_t max, double* link_bytes, int64_t* n) {
  if (sticky_) return sticky_;
  const int64_t cnt = std::min<int64_t>(max, (int64_t)prof_launch_link_.size());
  for (int64_t i = 0; i < cnt && link_bytes; ++i) link_bytes[i] = prof_launch_link_[i];
  if (n) *n = cnt;
  return HP_OK;
}

// Append the segments of a source covering global range [a, a+len): the acc
// slot `slot` of VW v (acc_of_vw) or w_global, wherever (which GPU) each part
// lives. Pointers are pre-offset so the launch's local index addresses them.
// Returns the number of segments added, or -1 if the table is full.
int Engine::add_segs(TickDesc& d, int64_t a, int64_t len, bool acc_of_vw, int v, int slot) {
  const int first = d.ns;
  for (int q = 0; q < G_; ++q) {
    const RankLayout& L = lay_[q];
    int64_t lo, hi;
    size_t off;
    if (acc_of_vw) {
      if (!L.has[v]) continue;
      lo = L.a[v];
      hi = L.a[v] + L.len[v];
      off = L.acc_off[v][slot];
    } else {
      lo = L.s0;
      hi = L.s1;
      off = L.wg_off;
    }
    const int64_t x0 = std::max(lo, a), x1 = std::min(hi, a + len);
    if (x0 >= x1) continue;
    if (d.ns == kMaxS) {
      d.ns = first;
      return -1;
    }
    // element i of the launch (global a + i) lives at buffer index a + i - lo
    const float* base = (const float*)(peer_[q] + off);
    d.s[d.ns].ptr = (const float*)((uintptr_t)base + (uintptr_t)((a - lo) * 4));
    d.s[d.ns].end = x1 - a;
    d.ns++;
  }
  // segments must come in increasing order of range (ranks hold increasing
  // ranges for w_global; a VW's stages are increasing in j but not in rank)
  std::sort(d.s + first, d.s + d.ns, [](const DSeg& x, const DSeg& y) { return x.end < y.end; });
  return d.ns - first;
}

hp_status Engine::flush() {
  if (sticky_) return sticky_;
  return dist_ ? flush_dist() : flush_local();
}

hp_status Engine::flush_local() {
  const bool strict = cfg_.local_semantics == HP_LOCAL_STRICT;
  TickDesc d;
  memset(&d, 0, sizeof d);
  // 1. completes (phase B)
  d.nc = (int)bc_.size();
  for (int j = 0; j < d.nc; ++j) {
    const BComplete& b = bc_[j];
    DComplete& c = d.c[j];
    c.acc = vw_[b.v].acc[b.slot];
    c.grad = b.grad;
    c.wl = nullptr;
    c.stash = convex_ ? vw_[b.v].stash[(b.p - 1) % Nm_] : nullptr;
    c.snap = b.snap ? vw_[b.v].snap : nullptr;
    c.v = (uint32_t)b.v;
    c.p = (uint32_t)b.p;
    c.flags = (b.first ? kFirst : kLoadAcc) | kStoreAcc | (b.snap ? kSnapAcc : 0u);
    c.neg_lr = neg_lr_of(b.v, b.p);
  }
  // 2. applies in commit order. The longest suffix whose waves were completed
  //    in this batch, in complete order, is applied straight from registers in
  //    phase B (u~ never reaches HBM); the rest are read from their acc slots in
  //    phase A, oldest first, overflow in apply-only launches before this one.
  size_t reg_from = ba_.size();
  int next_j = d.nc;
  while (reg_from > 0) {
    const BApply& a = ba_[reg_from - 1];
    int jj = -1;
    for (int j = 0; j < d.nc; ++j)
      if (bc_[j].v == a.v && bc_[j].wave_end && wave_of(bc_[j].p, U_) == a.c) jj = j;
    if (jj < 0 || jj >= next_j) break;
    next_j = jj;
    --reg_from;
  }
  // A memory-sourced apply must not read an acc slot this batch writes (phase A
  // runs before phase B): then the completes go out in a launch of their own.
  bool split = false;
  for (size_t k = 0; k < reg_from; ++k)
    for (int j = 0; j < d.nc; ++j)
      split |= bc_[j].v == ba_[k].v && bc_[j].wave_end && wave_of(bc_[j].p, U_) == ba_[k].c;
  if (split) {
    if (hp_status st = emit(d, begin_, n_)) return st;   // completes only: acc stored
    d.nc = 0;
    reg_from = ba_.size();
  }
  for (size_t k = reg_from; k < ba_.size(); ++k) {
    for (int j = 0; j < d.nc; ++j) {
      if (bc_[j].v == ba_[k].v && bc_[j].wave_end && wave_of(bc_[j].p, U_) == ba_[k].c) {
        d.c[j].flags |= kApplyNow;
        d.c[j].flags &= ~kStoreAcc;
      }
    }
  }
  size_t a0 = 0;
  while (reg_from - a0 > (size_t)kMaxA) {
    desc_splits_++;
    TickDesc pre;
    memset(&pre, 0, sizeof pre);
    for (int k = 0; k < kMaxA; ++k, ++a0) {
      pre.a[k].seg_begin = pre.ns;
      add_segs(pre, begin_, n_, true, ba_[a0].v, ba_[a0].slot);
      pre.a[k].seg_end = pre.ns;
    }
    pre.na = kMaxA;
    if (hp_status st = emit(pre, begin_, n_)) return st;
  }
  for (size_t k = a0; k < reg_from; ++k) {
    DApply& a = d.a[d.na++];
    a.seg_begin = d.ns;
    add_segs(d, begin_, n_, true, ba_[k].v, ba_[k].slot);
    a.seg_end = d.ns;
  }
  applied_ += (int64_t)ba_.size();
  apply_batches_ += ba_.empty() ? 0 : 1;
  // 3. w_local: pulled VWs and VWs whose folds are due now (phase D), or the
  //    single due fold of this batch's own complete, folded inline (phase B)
  for (int v = 0; v < N_; ++v) {
    VW& s = vw_[v];
    const bool pulled = std::find(bpull_.begin(), bpull_.end(), v) != bpull_.end();
    const bool hold = strict && s.at_gate;   // deferred to admission (Z3)
    if (!pulled && (hold || s.pending_folds.empty())) continue;
    std::vector<int64_t> folds;
    if (!hold) folds.swap(s.pending_folds);
    // the batch's own complete is the VW's only due fold (and, CONVEX, the
    // START that follows it): fold inline in phase B
    const bool tail_stash = folds.size() == 2 && folds[1] == -(folds[0] + Nm_);
    if (!pulled && (folds.size() == 1 || tail_stash) && folds[0] > 0) {
      int jj = -1;
      for (int j = 0; j < d.nc; ++j)
        if (bc_[j].v == v && bc_[j].p == folds[0]) jj = j;
      if (jj >= 0) {
        d.c[jj].flags |= kFoldInline | (tail_stash ? kStashAfter : 0u);
        d.c[jj].wl = s.wl;
        continue;
      }
    }
    size_t fi = 0;
    do {  // split a group whose folds overflow the descriptor
      if (d.ng == kMaxG || d.nf == kMaxF) {
        desc_splits_++;
        if (hp_status st = emit(d, begin_, n_)) return st;
        memset(&d, 0, sizeof d);
      }
      DGroup& g = d.g[d.ng++];
      g.wl = s.wl;
      g.pull = (pulled && fi == 0) ? 1 : 0;
      // w_global + the own unpushed aggregate (AT_LEAST; STRICT with F > 1),
      // stored in phase B if completed now
      g.partial = g.pull ? s.pull_partial : nullptr;
      g.f_begin = d.nf;
      for (; fi < folds.size() && d.nf < kMaxF; ++fi) fill_fold(d.f[d.nf++], v, folds[fi]);
      g.f_end = d.nf;
    } while (fi < folds.size());
  }
  bc_.clear();
  ba_.clear();
  bpull_.clear();
  phase_ = kNone;
  return emit(d, begin_, n_);
}

cudaEvent_t Engine::pool_event() {
  // Events are reused round-robin. A cudaStreamWaitEvent already enqueued keeps
  // the point the event was recorded at, so re-recording is safe -- except for
  // an event still stored as a dependency for a LATER wait (xacc_, xwl_, lastc_,
  // lastw_): those are skipped, so a stored dependency never silently moves.
  auto stored = [&](cudaEvent_t e) {
    for (const auto& x : xacc_)
      for (cudaEvent_t y : x)
        if (y == e) return true;
    for (const auto* vec : {&xwl_, &lastc_, &lastw_})
      for (cudaEvent_t y : *vec)
        if (y == e) return true;
    return false;
  };
  if (evpool_.size() >= 256) {
    for (size_t tries = 0; tries < evpool_.size(); ++tries) {
      cudaEvent_t e = evpool_[evnext_];
      evnext_ = (evnext_ + 1) % evpool_.size();
      if (!stored(e)) return e;
    }
  }
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  evpool_.push_back(e);
  return e;
}


int64_t Engine::local_len(int which) const {
  if (which == -1 || which == -2) return n_;
  return vw_[which].here ? vw_[which].len : 0;
}

hp_status Engine::flush_applies() {
  if (hp_status st = flush()) return st;
  if (pending_applies_.empty()) return HP_OK;
  for (auto& a : pending_applies_) ba_.push_back(a);
  pending_applies_.clear();
  return flush();
}

hp_status Engine::drain() {
  if (sticky_) return sticky_;
  if (capturing_ || graph_pending_) return fail(HP_ERR_STATE, "a captured graph has not been launched");
  if (hp_status st = flush_pending()) return st;
  if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "drain")) return st;
  return check_flag_err();
}

hp_status Engine::sync() {
  if (sticky_) return sticky_;
  if (capturing_ || graph_pending_) return fail(HP_ERR_STATE, "a captured graph has not been launched");
  for (auto& vp : ungated_) rec('S', vp.first, "START", vp.second, wave_of(vp.second, U_));
  ungated_.clear();
  if (hp_status st = flush_applies()) return st;
  if (hp_status st = join_exchange()) return st;
  if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "sync")) return st;
  return check_flag_err();
}

hp_status Engine::check_flag_err() {
  if (flag_err_) {                     // a K7 flag wait ran past its deadline
    int bad[8] = {0};
    // (on the context stream, never the legacy default stream: co-located
    // ranks share one CUDA context, see engine_dist.cpp finish_connect)
    if (hp_status st = check_cuda(cudaMemcpyAsync(bad, flag_err_, sizeof bad,
                                                  cudaMemcpyDeviceToHost, stream_),
                                  "flag error"))
      return st;
    if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "flag error")) return st;
    if (bad[0]) {
      sticky_ = HP_ERR_COMM;
      char buf[256];
      snprintf(buf, sizeof buf,
               "K7 readiness flag wait timed out (a rank stopped issuing barriers): rank %d "
               "waited for epoch %d, word held %d (wait %d of %d, %d signals; epochs: barrier "
               "%llu, apply %llu)",
               rank_, bad[1], bad[2], bad[3], bad[5], bad[4], (unsigned long long)epoch_,
               (unsigned long long)xepoch_);
      return fail(HP_ERR_COMM, buf);
    }
  }
  return HP_OK;
}

hp_status Engine::capture_begin() {
  if (sticky_) return sticky_;
  if (capturing_ || graph_pending_) return fail(HP_ERR_STATE, "a captured graph has not been launched");
  if (prof_on_) return fail(HP_ERR_STATE, "per-launch profiling is on: cannot capture");
  // (distributed contexts: a captured flag barrier would spin inside a graph
  // whose concurrency with the peers' work CUDA does not promise; they issue
  // their exchange directly)
  if (dist_) return fail(HP_ERR_STATE, "graph capture is for single-rank contexts");
  // earlier host-queued device work belongs to the stream before the graph
  if (hp_status st = flush_pending()) return st;
  if (int e = cudaStreamBeginCapture(stream_, cudaStreamCaptureModeRelaxed))
    return check_cuda(e, "cudaStreamBeginCapture");
  capturing_ = true;
  return HP_OK;
}

hp_status Engine::capture_end(bool ok, cudaGraphExec_t* exec) {
  if (!capturing_) return fail(HP_ERR_STATE, "not capturing");
  if (ok && !batch_.empty())
    if (flush_batch() != HP_OK) ok = false;
  batch_.clear();
  capturing_ = false;
  cudaGraph_t g = nullptr;
  const int e = cudaStreamEndCapture(stream_, &g);
  if (!ok) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    // the host state moved past device work that will never run
    sticky_ = HP_ERR_STATE;
    return sticky_;
  }
  if (e) return check_cuda(e, "cudaStreamEndCapture");
  const int e2 = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  if (e2) return check_cuda(e2, "cudaGraphInstantiate");
  graph_pending_ = true;
  return HP_OK;
}

// One multi-tick launch for the descriptors collected during a capture: they
// are uploaded now (synchronously, on a stream that is not captured) into a
// device buffer the graph owns, and the launch is recorded into the graph.
hp_status Engine::flush_batch() {
  if (batch_.empty()) return HP_OK;
  const size_t bytes = batch_.size() * sizeof(TickDescPad);
  void* dev = nullptr;
  if (cudaMalloc(&dev, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(HP_ERR_OOM, "tick batch allocation failed");
  }
  graph_bufs_.push_back(dev);
  if (!up_)
    if (int e = cudaStreamCreateWithFlags(&up_, cudaStreamNonBlocking)) return check_cuda(e, "stream");
  if (int e = cudaMemcpyAsync(dev, batch_.data(), bytes, cudaMemcpyHostToDevice, up_))
    return check_cuda(e, "tick batch upload");
  if (int e = cudaStreamSynchronize(up_)) return check_cuda(e, "tick batch upload");
  const int err = launch_multi_tick((const TickDescPad*)dev, (int)batch_.size(), n_, cfg_.grad_mode,
                                    m_ != nullptr, stream_);
  launches_++;
  batch_.clear();
  return check_cuda(err, "multi-tick kernel");
}

hp_status Engine::graph_launch(cudaGraphExec_t exec) {
  if (sticky_) return sticky_;
  if (!graph_pending_) return fail(HP_ERR_STATE, "no captured graph pending");
  graph_pending_ = false;
  return check_cuda(cudaGraphLaunch(exec, stream_), "cudaGraphLaunch");
}

// hp_launch_floor: device time per launch of n back-to-back empty kernels on
// the context stream, issued directly or as one captured graph (after one
// warm-up round of the same form).
hp_status Engine::launch_floor(int n, bool graph, float* us) {
  if (sticky_) return sticky_;
  if (capturing_ || graph_pending_) return fail(HP_ERR_STATE, "a captured graph has not been launched");
  if (n < 1 || !us) return fail(HP_ERR_INVALID, "n >= 1 and us needed");
  if (hp_status st = flush_pending()) return st;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaGraphExec_t exec = nullptr;
  int err = 0;
  if (graph) {
    cudaGraph_t g = nullptr;
    err = cudaStreamBeginCapture(stream_, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < n && !err; ++i) err = launch_empty(stream_);
    const int e2 = cudaStreamEndCapture(stream_, &g);
    if (!err) err = e2;
    if (!err) err = cudaGraphInstantiate(&exec, g, 0);
    if (g) cudaGraphDestroy(g);
  }
  float ms = 0.f;
  for (int rep = 0; rep < 2 && !err; ++rep) {     // rep 0 warms up
    cudaEventRecord(e0, stream_);
    if (graph) err = cudaGraphLaunch(exec, stream_);
    else
      for (int i = 0; i < n && !err; ++i) err = launch_empty(stream_);
    cudaEventRecord(e1, stream_);
    if (!err) err = cudaEventSynchronize(e1);
    if (!err) err = cudaEventElapsedTime(&ms, e0, e1);
  }
  if (exec) cudaGraphExecDestroy(exec);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err) return check_cuda(err, "launch floor");
  *us = 1e3f * ms / (float)n;
  return HP_OK;
}

hp_status Engine::read(int which, int64_t off, int64_t cnt, float* dst) {
  if (sticky_) return sticky_;
  if (which < -2 || which >= N_) return fail(HP_ERR_INVALID, "bad buffer id");
  if (which == -2 && !m_) return fail(HP_ERR_INVALID, "no momentum buffer");
  const int64_t len = local_len(which);
  if (off < 0 || cnt < 0 || off + cnt > len || (cnt && !dst)) return fail(HP_ERR_INVALID, "bad range");
  if (hp_status st = sync()) return st;
  const float* src = which == -1 ? wg_ : which == -2 ? m_ : vw_[which].wl;
  if (int e = cudaMemcpyAsync(dst, src + off, (size_t)cnt * 4, cudaMemcpyDeviceToHost, stream_))
    return check_cuda(e, "read");
  if (int e = cudaStreamSynchronize(stream_)) return check_cuda(e, "read");
  return HP_OK;
}

void Engine::stats(hp_stats* out) const {
  memset(out, 0, sizeof *out);
  out->commits = (int64_t)commit_.size();
  out->applied = applied_;
  out->launches = launches_;
  out->ticks = ticks;
  out->alg_bytes = alg_bytes_;
  for (int v = 0; v < N_ && v < 8; ++v) {
    out->wait_ticks[v] = vw_[v].wait;
    out->pulls[v] = vw_[v].pulls;
  }
  out->nvl_bytes = nvl_bytes_;
  out->lockstep_batches = lockstep_batches_;
  out->apply_batches = apply_batches_;
  out->desc_splits = desc_splits_;
}

hp_status Engine::profile_enable(bool on) {
  if (sticky_) return sticky_;
  if (capturing_ || graph_pending_) return fail(HP_ERR_STATE, "a captured graph has not been launched");
  prof_on_ = on;
  ev_used_ = 0;
  prof_bytes_ = 0;
  prof_launches_ = 0;
  prof_launch_bytes_.clear();
  prof_launch_sync_.clear();
  prof_launch_link_.clear();
  prof_launch_shape_.clear();
  prof_launch_stream_.clear();
  push_launch_.assign(N_, -1);
  sync_recs_.clear();
  return HP_OK;
}

hp_status Engine::profile_launches(int64_t max, float* ms, double* bytes, int32_t* shape,
                                   double* sync_bytes, float* start_ms, int64_t* n) {
  if (sticky_) return sticky_;
  if (hp_status st = join_exchange()) return st;
  if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "profile sync")) return st;
  const int64_t cnt = std::min<int64_t>(max, (int64_t)prof_launch_bytes_.size());
  for (int64_t i = 0; i < cnt; ++i) {
    float t = 0;
    if (int e = cudaEventElapsedTime(&t, ev_[2 * i], ev_[2 * i + 1])) return check_cuda(e, "elapsed");
    if (ms) ms[i] = t;
    if (bytes) bytes[i] = prof_launch_bytes_[i];
    if (shape) shape[i] = prof_launch_shape_[i];
    if (sync_bytes) sync_bytes[i] = prof_launch_sync_[i];
    if (start_ms) {   // launch start relative to the first profiled launch (any stream)
      float t0 = 0;
      if (int e = cudaEventElapsedTime(&t0, ev_[0], ev_[2 * i])) return check_cuda(e, "elapsed");
      start_ms[i] = t0;
    }
  }
  if (n) *n = cnt;
  return HP_OK;
}

hp_status Engine::profile_read(double* ms, double* bytes, int64_t* launches) {
  if (sticky_) return sticky_;
  if (hp_status st = join_exchange()) return st;
  if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "profile sync")) return st;
  double tot = 0;
  for (size_t i = 0; i + 1 < ev_used_; i += 2) {
    float t = 0;
    if (int e = cudaEventElapsedTime(&t, ev_[i], ev_[i + 1])) return check_cuda(e, "elapsed");
    tot += t;
  }
  if (ms) *ms = tot;
  if (bytes) *bytes = prof_bytes_;
  if (launches) *launches = prof_launches_;
  return HP_OK;
}

}  // namespace hp

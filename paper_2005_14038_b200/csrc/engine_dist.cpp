// engine_dist.cpp -- the distributed placements of the WSP engine (world > 1):
// the per-batch exchange (accumulation streams, PS applies over NVLink, pulls),
// the lockstep transports (NCCL, NVLS), and the set-up (IPC or symmetric
// arenas, communicator, streams). The protocol state and the single-rank
// batch live in engine.cpp; see engine.h.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine.h"

namespace hp {

// Distributed flush (world > 1). Replicated on every rank with identical
// decisions, so every rank issues the same barriers. Streams (row a9,
// overlap): each local VW's accumulation runs on its own stream; barriers,
// applies and pulls run on the exchange stream xs_, which waits only for the
// accumulation launches whose results it reads, and a VW's stream waits only
// for the exchange ops that touched that VW's buffers.
//   1. per local VW: its complete (acc always stored: peers read it) with an
//      inline fold, or its fold-only group, on the VW's stream;
//   2. if the batch applies pushes: xs_ waits for the pushing VWs' streams ->
//      BARRIER (every rank's pushed u~ complete; earlier pulls of w_global done
//      everywhere) -> apply launch(es) over this rank's PS shard reading every
//      pushed u~ slice from the GPU that holds it (NVLink loads inside the
//      kernel, commit order) -> BARRIER (w_global final; acc slots reusable);
//   3. pulls on xs_: w_local(v) of each local stage <- w_global read from the
//      shard owners (NVLink loads), then the VW's due folds.
hp_status Engine::flush_dist() {
  fork_streams();
  std::vector<bool> pulled(N_, false);
  for (int v : bpull_) pulled[v] = true;
  if (hp_status st = dist_accumulate(pulled)) return st;
  // ---- lockstep batches under HP_XPORT_NCCL / NVLS ------------------------
  const int lslot = lockstep_slot();
  if (lslot >= 0) return flush_lockstep(lslot);
  std::vector<Prim> prims;
  bool fuse_pull = false;
  if (hp_status st = dist_apply(&prims, &fuse_pull)) return st;
  if (hp_status st = dist_pull(prims, fuse_pull)) return st;
  bc_.clear();
  ba_.clear();
  bpull_.clear();
  phase_ = kNone;
  return HP_OK;
}

// Step 1: each local VW's completes and due folds on its own streams.
hp_status Engine::dist_accumulate(const std::vector<bool>& pulled) {
  const bool strict = cfg_.local_semantics == HP_LOCAL_STRICT;
  // ---- 1. accumulation, one launch per local VW on its own stream ----------
  for (int v = 0; v < N_; ++v) {
    VW& s = vw_[v];
    if (!s.here) {
      if (!pulled[v] && !(strict && s.at_gate)) s.pending_folds.clear();  // peers' work
      continue;
    }
    TickDesc d;
    memset(&d, 0, sizeof d);
    int cslot[kMaxC];
    for (const BComplete& b : bc_) {
      if (b.v != v) continue;
      cslot[d.nc] = b.slot;
      DComplete& c = d.c[d.nc++];
      c.acc = s.acc[b.slot];
      c.grad = b.grad;                  // EXTERNAL: this rank's stage of u's gradient
      c.wl = nullptr;
      c.stash = convex_ ? s.stash[(b.p - 1) % Nm_] : nullptr;
      c.snap = b.snap ? s.snap : nullptr;
      c.v = (uint32_t)b.v;
      c.p = (uint32_t)b.p;
      c.flags = (b.first ? kFirst : kLoadAcc) | kStoreAcc | (b.snap ? kSnapAcc : 0u);
      c.neg_lr = neg_lr_of(b.v, b.p);
    }
    const bool hold = strict && s.at_gate;
    std::vector<int64_t> folds;
    if (!pulled[v] && !hold) folds.swap(s.pending_folds);
    if (d.nc == 0 && folds.empty()) continue;
    auto wait_clear = [](cudaStream_t st, cudaEvent_t& e) {
      if (e) cudaStreamWaitEvent(st, e, 0);
      e = nullptr;
    };
    cudaStream_t fst = vs_[v];          // stream of the w_local folds
    // (CONVEX: a complete reads the stash slot the folds' STASH ops write, so
    // acc and folds stay in one launch)
    if (split_folds_ && !convex_) {
      // acc part now (its slot is free once the exchange that read it is done)
      if (d.nc) {
        for (int j = 0; j < d.nc; ++j) wait_clear(vs_[v], xacc_[v][cslot[j]]);
        if (hp_status st = emit(d, s.a0, s.len, vs_[v], ablocks_)) return st;
        lastc_[v] = pool_event();
        cudaEventRecord(lastc_[v], vs_[v]);
        memset(&d, 0, sizeof d);
      }
      if (folds.empty()) continue;
      fst = fs_[v];                     // folds after the pull that rewrote w_local
      wait_clear(fst, xwl_[v]);
      if (lastw_[v]) cudaStreamWaitEvent(fst, lastw_[v], 0);
      // EXTERNAL gradients: a fold reads the gradient slot its minibatch's
      // host copy filled on the accumulation stream -- after that copy (the
      // acc launches follow their copies on vs_, so after the last of them)
      if (cfg_.grad_mode == HP_GRAD_EXTERNAL && lastc_[v]) cudaStreamWaitEvent(fst, lastc_[v], 0);
      // a single FOLD is the inline fold of a complete without its
      // acc part: it takes the lean completes-only instance (4 chunks per
      // thread, 4 CTAs/SM) instead of the group path, whose 2-chunk / 3-CTA
      // shape leaves a one-buffer launch latency-bound (HP_FOLD_LEAN=0: group)
      static const int fold_lean = getenv("HP_FOLD_LEAN") ? atoi(getenv("HP_FOLD_LEAN")) : 1;
      if (fold_lean && folds.size() == 1 && folds[0] > 0) {
        DComplete& c = d.c[d.nc++];
        c.wl = s.wl;
        c.grad = fold_grad(v, folds[0]);
        c.v = (uint32_t)v;
        c.p = (uint32_t)folds[0];
        c.flags = kFoldInline;
        c.neg_lr = neg_lr_of(v, folds[0]);
        folds.clear();
      }
    } else {
      for (int j = 0; j < d.nc; ++j) wait_clear(vs_[v], xacc_[v][cslot[j]]);
      wait_clear(vs_[v], xwl_[v]);
      if (lastw_[v]) cudaStreamWaitEvent(vs_[v], lastw_[v], 0);
      const bool tail_stash = folds.size() == 2 && folds[1] == -(folds[0] + Nm_);
      if ((folds.size() == 1 || tail_stash) && d.nc == 1 && (int64_t)d.c[0].p == folds[0]) {
        d.c[0].flags |= kFoldInline | (tail_stash ? kStashAfter : 0u);
        d.c[0].wl = s.wl;
        folds.clear();
      }
    }
    size_t fi = 0;
    while (fi < folds.size()) {
      if (d.ng == kMaxG || d.nf == kMaxF) {
        desc_splits_++;
        if (hp_status st = emit(d, s.a0, s.len, fst, ablocks_)) return st;
        memset(&d, 0, sizeof d);
      }
      DGroup& g = d.g[d.ng++];
      g.wl = s.wl;
      g.pull = 0;
      g.f_begin = d.nf;
      for (; fi < folds.size() && d.nf < kMaxF; ++fi) {
        fill_fold(d.f[d.nf++], v, folds[fi]);
      }
      g.f_end = d.nf;
    }
    if (hp_status st = emit(d, s.a0, s.len, fst, ablocks_)) return st;
    cudaEvent_t e = pool_event();
    cudaEventRecord(e, fst);
    if (fst == vs_[v]) lastc_[v] = e;   // (fs_ launches write no acc slot)
    lastw_[v] = e;
  }
  return HP_OK;
}

// Step 2: BARRIER -> the applies of this rank's PS shard (NVLink loads of the
// pushed u~; owner-side pull stores) -> BARRIER, on the exchange stream.
hp_status Engine::dist_apply(std::vector<Prim>* prims_out, bool* fuse_out) {
  const bool strict = cfg_.local_semantics == HP_LOCAL_STRICT;
  // ---- 2. exchange stream: wait only for the producers it reads ------------
  auto xs_wait = [&](int v) {
    if (vw_[v].here && lastc_[v]) cudaStreamWaitEvent(xs_, lastc_[v], 0);
  };
  auto xs_wait_wl = [&](int v) {      // a pull rewrites w_local: after its folds
    if (vw_[v].here && lastw_[v]) cudaStreamWaitEvent(xs_, lastw_[v], 0);
  };
  // Owner-side pull (STRICT: the pull is the copy w_local = w_global): the
  // last apply launch also stores the final w_global of this rank's shard into
  // every pulled VW's w_local slice, wherever it lives (NVLink stores, under the
  // loads of the applies); the post-apply barrier publishes them. HP_PULL_PUSH=0
  // keeps the separate reader-side pull launches.
  // One target per (GPU, stage range): the first pulled VW there (its
  // "primary"); the other pulled VWs of that GPU and range copy it locally
  // afterwards (fan-out, as the reader-side pull reads a remote shard once).

  std::vector<Prim>& prims = *prims_out;
  prims.clear();
  for (int v : bpull_)
    for (int q = 0; q < G_; ++q) {
      const RankLayout& L = lay_[q];
      if (!L.has[v]) continue;
      bool seen = false;
      for (const Prim& pr : prims) seen |= pr.q == q && pr.a == L.a[v] && pr.len == L.len[v];
      if (!seen) prims.push_back({q, L.a[v], L.len[v], v});
    }
  std::vector<DStore> ptargets;
  for (const Prim& pr : prims) {
    const RankLayout& L = lay_[pr.q];
    const int64_t x0 = std::max(pr.a, begin_), x1 = std::min(pr.a + pr.len, begin_ + n_);
    if (x0 >= x1) continue;
    float* base = (float*)(peer_[pr.q] + L.wl_off[pr.v]);
    ptargets.push_back({base + (begin_ - pr.a), x0 - begin_, x1 - begin_});   // i -> [begin_+i-a]
  }
  // every rank must take the same decision: fuse only if no owner's shard
  // meets more than kMaxP targets (shards may be uneven, hp_config.ps_bounds)
  size_t max_targets = 0;
  for (int o = 0; o < G_; ++o) {
    size_t cnt = 0;
    for (const Prim& pr : prims)
      cnt += std::max(pr.a, shard_b_[o]) < std::min(pr.a + pr.len, shard_b_[o + 1]) ? 1 : 0;
    max_targets = std::max(max_targets, cnt);
  }
  const bool fuse_pull = *fuse_out = push_pull_ && strict && U_ == Nm_ && !ba_.empty() &&
                                     !bpull_.empty() && max_targets <= (size_t)kMaxP;
  if (push_pull_ && strict && U_ == Nm_ && !ba_.empty() && !bpull_.empty() && !fuse_pull)
    desc_splits_++;                   // owner-side pull refused: too many targets
  // NVLink traffic of this rank's links while every owner runs its apply
  // launch at once (the barrier aligns them): the ũ slices it loads from peers
  // and the owner-side pull stores it receives (in), what peers load from it and
  // the stores it sends (out); reported per direction as max(in, out)
  double x_in = 0, x_out = 0;
  auto flow = [&](int from, int to, double bytes) {
    if (from == to) return;
    if (to == rank_) x_in += bytes;
    if (from == rank_) x_out += bytes;
  };
  for (int o = 0; o < G_ && !ba_.empty(); ++o) {
    const int64_t s0 = shard_b_[o], s1 = shard_b_[o + 1];
    for (const BApply& a : ba_)
      for (int g = 0; g < G_; ++g) {
        const RankLayout& L = lay_[g];
        if (!L.has[a.v]) continue;
        const int64_t x0 = std::max(L.a[a.v], s0), x1 = std::min(L.a[a.v] + L.len[a.v], s1);
        if (x1 > x0) flow(g, o, 4.0 * (double)(x1 - x0));
      }
    if (fuse_pull)
      for (const Prim& pr : prims) {
        const int64_t x0 = std::max(pr.a, s0), x1 = std::min(pr.a + pr.len, s1);
        if (x1 > x0) flow(o, pr.q, 4.0 * (double)(x1 - x0));
      }
  }
  int n_apply_launches = 0;
  for (size_t k2 = 0; k2 < ba_.size(); k2 += kMaxA) ++n_apply_launches;
  if (n_apply_launches > 1) desc_splits_ += n_apply_launches - 1;
  const double x_link = n_apply_launches ? std::max(x_in, x_out) / n_apply_launches : 0.0;
  // ranks this batch involves: every stage of a pushing VW (its u~ is read by
  // every owner; its acc slot is reused only after all owners read it), every
  // stage of a pulled VW (its w_local is written by every owner, after its own
  // folds), and the ranks that read w_global shards since the last apply (WAR)
  std::vector<char> inv(G_, 0);
  for (const BApply& a : ba_)
    for (int q = 0; q < G_; ++q) inv[q] |= lay_[q].has[a.v];
  for (int v : bpull_)
    for (int q = 0; q < G_; ++q) inv[q] |= lay_[q].has[v];
  for (int q = 0; q < G_; ++q) inv[q] |= readers_[q];
  const bool p2p = p2p_ && flag_barrier_;
  if (!ba_.empty()) {
    for (const BApply& a : ba_) xs_wait(a.v);
    for (int v : bpull_) {
      xs_wait(v);
      xs_wait_wl(v);
    }
    const uint64_t ep = p2p ? ++xepoch_ : 0;
    if (p2p) {
      // ARRIVE: an involved rank announces its producers are done to every
      // owner; every owner (all ranks) waits for the involved ranks only
      std::vector<unsigned long long*> sig;
      std::vector<const unsigned long long*> wait;
      if (inv[rank_])
        for (int q = 0; q < G_; ++q) sig.push_back(flag_word(q, 1, rank_));
      for (int q = 0; q < G_; ++q)
        if (inv[q]) wait.push_back(flag_word(rank_, 1, q));
      if (hp_status st = flag_ops(xs_, sig, wait, ep)) return st;
    } else if (hp_status st = xbarrier()) {
      return st;
    }
    size_t k = 0;
    while (k < ba_.size()) {
      TickDesc d;
      memset(&d, 0, sizeof d);
      while (k < ba_.size() && d.na < kMaxA) {
        const int b = d.ns;
        if (add_segs(d, begin_, n_, true, ba_[k].v, ba_[k].slot) < 0) {
          desc_splits_++;               // segment table full: the rest in a later launch
          break;
        }
        d.a[d.na].seg_begin = b;
        d.a[d.na].seg_end = d.ns;
        d.na++;
        ++k;
      }
      if (fuse_pull && k == ba_.size())
        for (const DStore& t : ptargets) d.pd[d.np++] = t;
      if (hp_status st = emit(d, begin_, n_, xs_, xblocks_, x_link)) return st;
    }
    applied_ += (int64_t)ba_.size();
    apply_batches_++;
    if (p2p) {
      // DONE: every owner tells every rank its applies (and owner-side pull
      // stores) are complete; an involved rank waits for every owner -- an
      // uninvolved one does not wait at all (a later reader-side pull of it
      // waits on the same words)
      std::vector<unsigned long long*> sig;
      std::vector<const unsigned long long*> wait;
      for (int q = 0; q < G_; ++q) sig.push_back(flag_word(q, 2, rank_));
      if (inv[rank_])
        for (int q = 0; q < G_; ++q) wait.push_back(flag_word(rank_, 2, q));
      if (hp_status st = flag_ops(xs_, sig, wait, ep)) return st;
      last_apply_epoch_ = ep;
      std::fill(readers_.begin(), readers_.end(), 0);
    } else if (hp_status st = xbarrier()) {
      return st;
    }
    cudaEvent_t e = pool_event();       // acc slots read by the applies are free
    cudaEventRecord(e, xs_);
    for (const BApply& a : ba_)
      if (vw_[a.v].here) xacc_[a.v][a.slot] = e;
  } else {
    for (int v : bpull_) {
      xs_wait(v);
      xs_wait_wl(v);
    }
  }
  return HP_OK;
}

// Step 3: the pulls -- the fan-out copies and folds after an owner-side pull,
// or reader-side pull launches.
hp_status Engine::dist_pull(const std::vector<Prim>& prims, bool fuse_pull) {
  const bool strict = cfg_.local_semantics == HP_LOCAL_STRICT;
  // ---- 3. pulls: per local stage range one launch reads w_global from the
  //      shard owners once (into registers) and writes every pulled w_local of
  //      that range, each followed by its own due folds ----------------------
  std::vector<std::pair<int64_t, int64_t>> pranges;
  for (int v : bpull_) {
    VW& s = vw_[v];
    if (!s.here) {
      s.pending_folds.clear();
      continue;
    }
    if (std::find(pranges.begin(), pranges.end(), std::make_pair(s.a0, s.len)) == pranges.end())
      pranges.push_back({s.a0, s.len});
  }
  if (fuse_pull) {   // the owners stored w_global into the primaries' w_local
    note_pulls(bpull_);                  // (wave-sync latency: ends with this apply)
    for (auto& rg : pranges) {
      int prim = -1;
      for (const Prim& pr : prims)
        if (pr.q == rank_ && pr.a == rg.first && pr.len == rg.second) prim = pr.v;
      const int64_t ov = std::max<int64_t>(
          0, std::min(rg.first + rg.second, begin_ + n_) - std::max(rg.first, begin_));
      nvl_bytes_ += 4.0 * (double)(rg.second - ov);   // received from the other owners
      // the other pulled VWs of this range copy the primary (groups before the
      // primary's own folds: the kernel runs groups in order per element),
      // then every VW's due folds
      std::vector<int> order;
      for (int v : bpull_)
        if (vw_[v].here && vw_[v].a0 == rg.first && vw_[v].len == rg.second && v != prim)
          order.push_back(v);
      order.push_back(prim);
      TickDesc d;
      memset(&d, 0, sizeof d);
      for (int v : order) {
        VW& s = vw_[v];
        std::vector<int64_t> folds;
        folds.swap(s.pending_folds);
        if (v == prim && folds.empty()) continue;
        size_t fi = 0;
        bool first_part = true;
        do {
          if (d.ng == kMaxG || d.nf == kMaxF || d.ns == kMaxS) {
            desc_splits_++;
            if (hp_status st = emit(d, rg.first, rg.second, xs_, xblocks_)) return st;
            memset(&d, 0, sizeof d);
          }
          DGroup& g = d.g[d.ng++];
          g.wl = s.wl;
          g.pull = 0;
          if (first_part && v != prim) {       // base = the primary's pulled w_local
            g.pull = 2;
            g.seg_begin = d.ns;
            d.s[d.ns].ptr = vw_[prim].wl;
            d.s[d.ns].end = rg.second;
            d.ns++;
            g.seg_end = d.ns;
          }
          first_part = false;
          g.f_begin = d.nf;
          for (; fi < folds.size() && d.nf < kMaxF; ++fi) {
            fill_fold(d.f[d.nf++], v, folds[fi]);
          }
          g.f_end = d.nf;
        } while (fi < folds.size());
      }
      if (d.ng)
        if (hp_status st = emit(d, rg.first, rg.second, xs_, xblocks_)) return st;
    }
    pranges.clear();
  }
  // reader-side pull traffic of this rank's links while every rank pulls: the
  // remote shards its stage ranges read (in) and what the other GPUs' ranges
  // read from its shard (out)
  double r_link = 0;
  if (!pranges.empty()) {
    double r_in = 0, r_out = 0;
    for (int g = 0; g < G_; ++g) {
      std::vector<std::pair<int64_t, int64_t>> rr;
      for (int v : bpull_) {
        const RankLayout& L = lay_[g];
        if (!L.has[v]) continue;
        auto key = std::make_pair(L.a[v], L.len[v]);
        if (std::find(rr.begin(), rr.end(), key) == rr.end()) rr.push_back(key);
      }
      for (auto& r : rr)
        for (int o = 0; o < G_; ++o) {
          if (o == g) continue;
          const int64_t x0 = std::max(r.first, shard_b_[o]);
          const int64_t x1 = std::min(r.first + r.second, shard_b_[o + 1]);
          if (x1 <= x0) continue;
          if (g == rank_) r_in += 4.0 * (double)(x1 - x0);
          if (o == rank_) r_out += 4.0 * (double)(x1 - x0);
        }
    }
    r_link = std::max(r_in, r_out) / (double)pranges.size();
  }
  if (p2p_ && flag_barrier_ && !fuse_pull && !bpull_.empty()) {
    // reader-side pulls read every owner's w_global: after its last apply
    // (this rank may not have been involved in that batch), and the readers
    // hold off the owners' next apply (readers_, replicated on every rank)
    if (!pranges.empty() && last_apply_epoch_ > 0) {
      std::vector<const unsigned long long*> wait;
      for (int q = 0; q < G_; ++q) wait.push_back(flag_word(rank_, 2, q));
      if (hp_status st = flag_ops(xs_, {}, wait, last_apply_epoch_)) return st;
    }
    for (int v : bpull_)
      for (int q = 0; q < G_; ++q) readers_[q] |= lay_[q].has[v];
  }
  for (auto& rg : pranges) {
    TickDesc d;
    auto fresh = [&]() {
      memset(&d, 0, sizeof d);
      d.wgs_begin = d.ns;
      add_segs(d, rg.first, rg.second, false, 0, 0);
      d.wgs_end = d.ns;
    };
    fresh();
    for (int v : bpull_) {
      VW& s = vw_[v];
      if (!s.here || s.a0 != rg.first || s.len != rg.second) continue;
      std::vector<int64_t> folds;
      folds.swap(s.pending_folds);
      size_t fi = 0;
      bool first_part = true;
      do {
        if (d.ng == kMaxG || d.nf == kMaxF) {
          desc_splits_++;
          if (hp_status st = emit(d, rg.first, rg.second, xs_, xblocks_, r_link)) return st;
          fresh();
        }
        DGroup& g = d.g[d.ng++];
        g.wl = s.wl;
        g.partial = nullptr;
        g.pull = first_part ? 1 : 0;     // 1: base = the w_global registers
        if (first_part) g.partial = s.pull_partial;
        first_part = false;
        g.f_begin = d.nf;
        for (; fi < folds.size() && d.nf < kMaxF; ++fi) {
          fill_fold(d.f[d.nf++], v, folds[fi]);
        }
        g.f_end = d.nf;
      } while (fi < folds.size());
    }
    if (hp_status st = emit(d, rg.first, rg.second, xs_, xblocks_, r_link)) return st;
  }
  if (!bpull_.empty()) {
    cudaEvent_t e = pool_event();       // w_local of the pulled VWs is written
    cudaEventRecord(e, xs_);
    for (int v : bpull_)
      if (vw_[v].here) {
        xwl_[v] = e;
        lastw_[v] = nullptr;              // ordered behind e
        // the pull read a partial aggregate (AT_LEAST; STRICT with F > 1): the
        // acc slot of the open clock or, STRICT, the snapshot taken at the gate.
        // Completes that rewrite it wait for e. The snapshot is rewritten by a
        // complete of a later clock, whatever its slot: every slot waits then
        // (xs_ is in order, so e covers the events it replaces).
        const float* part = vw_[v].pull_partial;
        if (part && part == vw_[v].snap) {
          for (auto& x : xacc_[v]) x = e;
        } else if (part || !strict) {
          xacc_[v][vw_[v].c_local % R_] = e;
        }
      }
  }
  return HP_OK;
}

// A lockstep batch: one full-replica VW per GPU (N = G, span 1, so VW v lives
// on GPU v at identical arena offsets), SGD, and the batch applies exactly one
// push of the same wave c from every VW, and pulls either no VW or every VW
// (STRICT: the pull is the copy w_local = w_global). Returns the acc slot of
// wave c, or -1 (the batch takes the PEER path).
int Engine::lockstep_slot() const {
  // (F > 1: a STRICT pull adds the open clock's aggregate, which the
  // collective copy w_local = w_global does not)
  if (cfg_.transport == HP_XPORT_PEER || !dist_ || G_ != N_ || span_ != 1 || m_ || U_ != Nm_)
    return -1;
  if (cfg_.transport == HP_XPORT_NVLS && !mc_) return -1;
  if ((int)ba_.size() != N_) return -1;
  std::vector<char> seen(N_, 0);
  for (const BApply& a : ba_) {
    if (a.c != ba_[0].c || seen[a.v]) return -1;
    seen[a.v] = 1;
  }
  if (!bpull_.empty()) {
    if ((int)bpull_.size() != N_ || cfg_.local_semantics != HP_LOCAL_STRICT) return -1;
    std::vector<char> pulled(N_, 0);
    for (int v : bpull_) {
      if (pulled[v]) return -1;
      pulled[v] = 1;
    }
  }
  return ba_[0].slot;
}

// Exchange of a lockstep batch (PAPER.md P:928-929 apply, P:949 pull): the N
// pushed u~ of wave c are summed per PS shard and applied once, then every VW
// pulls the new w_global.
//   NVLS: BARRIER -> one kernel per owner: multimem.ld_reduce of its shard of
//         every GPU's acc slot, w_global += sum, multimem.st into every GPU's
//         w_local -> BARRIER.
//   NCCL: grouped ncclReduce (reduce-scatter) of the acc slot into the staging
//         shard -> apply launch -> grouped ncclBroadcast (all-gather) of the
//         w_global shards into w_local.
// Then each pulled VW's due folds (the backlog, Z17) on the exchange stream.
hp_status Engine::flush_lockstep(int slot) {
  for (const BApply& a : ba_)
    if (vw_[a.v].here && lastc_[a.v]) cudaStreamWaitEvent(xs_, lastc_[a.v], 0);
  for (int v : bpull_) {
    if (vw_[v].here && lastc_[v]) cudaStreamWaitEvent(xs_, lastc_[v], 0);
    if (vw_[v].here && lastw_[v]) cudaStreamWaitEvent(xs_, lastw_[v], 0);
  }
  const int me = rank_;             // VW `me` lives on this GPU
  VW& s = vw_[me];
  const bool pull = !bpull_.empty();
  const RankLayout& L = lay_[me];
  const double P = (double)cfg_.nparams, n = (double)n_;
  if (cfg_.transport == HP_XPORT_NVLS) {
    if (hp_status st = xbarrier()) return st;
    // HP_NVLS_SPLIT < 100: the tail of the shard goes through the peer path
    // (NVLink loads of the u~ slices + owner-side stores into every w_local)
    // on a second exchange stream, concurrently with the multicast kernel
    const int64_t n1 = nvls_split_ >= 100 ? n_ : (n_ * nvls_split_ / 100) / 32 * 32;
    cudaEvent_t peer_done = nullptr;
    if (n1 < n_) {
      cudaEvent_t e0 = pool_event();
      cudaEventRecord(e0, xs_);
      cudaStreamWaitEvent(xs2_, e0, 0);
      TickDesc t;
      memset(&t, 0, sizeof t);
      for (const BApply& a : ba_) {
        const int b = t.ns;
        add_segs(t, begin_ + n1, n_ - n1, true, a.v, a.slot);
        t.a[t.na].seg_begin = b;
        t.a[t.na].seg_end = t.ns;
        t.na++;
      }
      if (pull)
        for (int q = 0; q < G_; ++q)
          t.pd[t.np++] = {(float*)(peer_[q] + lay_[q].wl_off[q]) + begin_ + n1, 0, n_ - n1};
      const double tl = 4.0 * (double)(n_ - n1) * (G_ - 1) * (pull ? 2.0 : 1.0);
      if (hp_status st = emit(t, begin_ + n1, n_ - n1, xs2_, xblocks_, tl)) return st;
      peer_done = pool_event();
      cudaEventRecord(peer_done, xs2_);
    }
    NvlsDesc d;
    memset(&d, 0, sizeof d);
    d.n = n1;
    d.wg = wg_;
    d.mc_acc = (const float*)(mc_ + L.acc_off[me][slot]) + begin_;
    d.mc_wl = pull ? (float*)(mc_ + L.wl_off[me]) + begin_ : nullptr;
    d.G = G_;
    for (int q = 0; q < G_; ++q) {
      d.src[q] = (const float*)(peer_[q] + lay_[q].acc_off[q][slot]) + begin_;
      d.dst[q] = (float*)(peer_[q] + lay_[q].wl_off[q]) + begin_;
    }
    static const int nvls_dyn = getenv("HP_NVLS_DYN") ? atoi(getenv("HP_NVLS_DYN")) : 1;
    if (nvls_dyn) tile_slot(xs_, &d.ctr, &d.done);
    const double fr = n_ > 0 ? (double)n1 / (double)n_ : 0.0;   // multicast share
    const double bytes = 4.0 * (double)n1 * (2 + G_ + (pull ? G_ : 0));
    stress(xs_);
    prof_begin(xs_);
    const int err = launch_nvls(d, xs_, xblocks_);
    // per GPU and direction: its acc replica served to every owner's reduction
    // (4P through the switch) + the multicast store (4n out / 4P in)
    prof_end(xs_, bytes, bytes, (N_ << 8) | (pull ? (int)(1u << 31) : 0),
             (4.0 * P + (pull ? 4.0 * n : 0.0)) * fr);
    if (pull) note_pulls(bpull_);
    if (n1 > 0) launches_++;
    alg_bytes_ += bytes;
    nvl_bytes_ += (4.0 * n + (pull ? 4.0 * (P - n) : 0.0)) * fr;
    if (hp_status st = check_cuda(err, "nvls kernel")) return st;
    if (peer_done) cudaStreamWaitEvent(xs_, peer_done, 0);
    if (hp_status st = xbarrier()) return st;
  } else {
    float* x = (float*)((char*)arena_ + L.x_off);
    // the collectives are profiled like launches: bytes = what they read and
    // write in this rank's HBM (send buffer + received data)
    int64_t smax = 0;
    for (int q = 0; q < G_; ++q) smax = std::max(smax, shard_b_[q + 1] - shard_b_[q]);
    // the NCCL transport's default shards (ceil split) are smax long but the
    // last: the equal-count collectives run on the padded buffers; other
    // bounds (hp_config.ps_bounds) take the grouped per-shard form
    bool equal = true;
    for (int q = 0; q + 1 < G_; ++q) equal &= shard_b_[q + 1] - shard_b_[q] == smax;
    prof_begin(xs_);
    if ((equal ? comm_->reduce_scatter(s.acc[slot], x, smax, xs_)
               : comm_->reduce_scatter_v(s.acc[slot], x, shard_b_.data(), xs_)) != 0)
      return fail(HP_ERR_COMM, comm_->error());
    prof_end(xs_, 4.0 * (P + n), 4.0 * (P + n), (1 << 8) | (127 << 24), 4.0 * n * (G_ - 1));
    TickDesc d;
    memset(&d, 0, sizeof d);
    d.s[0].ptr = x;
    d.s[0].end = n_;
    d.ns = 1;
    d.a[0].seg_begin = 0;
    d.a[0].seg_end = 1;
    d.na = 1;
    if (hp_status st = emit(d, begin_, n_, xs_)) return st;
    if (pull) {
      prof_begin(xs_);
      if ((equal ? comm_->all_gather(wg_, s.wl, smax, xs_)
                 : comm_->all_gather_v(wg_, s.wl, shard_b_.data(), xs_)) != 0)
        return fail(HP_ERR_COMM, comm_->error());
      prof_end(xs_, 4.0 * (P + n), 4.0 * (P + n), (1 << 16) | (127 << 24) | (int)(1u << 31),
               4.0 * (P - n));
      note_pulls(bpull_);
    }
    nvl_bytes_ += 4.0 * n * (G_ - 1) + (pull ? 4.0 * (P - n) : 0.0);
  }
  applied_ += (int64_t)ba_.size();
  lockstep_batches_++;
  apply_batches_++;
  for (int v : bpull_) {
    VW& t = vw_[v];
    std::vector<int64_t> folds;
    folds.swap(t.pending_folds);
    if (!t.here || folds.empty()) continue;
    size_t fi = 0;
    while (fi < folds.size()) {
      TickDesc d;
      memset(&d, 0, sizeof d);
      while (fi < folds.size() && d.ng < kMaxG && d.nf < kMaxF) {
        DGroup& g = d.g[d.ng++];
        g.wl = t.wl;
        g.pull = 0;
        g.f_begin = d.nf;
        for (; fi < folds.size() && d.nf < kMaxF; ++fi) {
          fill_fold(d.f[d.nf++], v, folds[fi]);
        }
        g.f_end = d.nf;
      }
      if (hp_status st = emit(d, t.a0, t.len, xs_)) return st;
    }
  }
  cudaEvent_t e = pool_event();       // acc slots free, w_local of the pullers written
  cudaEventRecord(e, xs_);
  for (const BApply& a : ba_)
    if (vw_[a.v].here) xacc_[a.v][a.slot] = e;
  for (int v : bpull_)
    if (vw_[v].here) {
      xwl_[v] = e;
      lastw_[v] = nullptr;
    }
  bc_.clear();
  ba_.clear();
  bpull_.clear();
  phase_ = kNone;
  return HP_OK;
}

unsigned long long* Engine::flag_word(int q, int kind, int src) const {
  return (unsigned long long*)(peer_[q] + lay_[q].flag_off) + (size_t)kind * G_ + src;
}

// Flag publications and waits on stream st (chunks of 8), profiled like the
// barrier (shape nf = 126).
hp_status Engine::flag_ops(cudaStream_t st, std::vector<unsigned long long*> sig,
                           std::vector<const unsigned long long*> wait, uint64_t val) {
  size_t i = 0, j = 0;
  while (i < sig.size() || j < wait.size()) {
    FlagOps fo;
    memset(&fo, 0, sizeof fo);
    fo.val = val;
    fo.err = flag_err_;
    fo.timeout_ns = flag_timeout_ns_;
    for (; i < sig.size() && fo.nsig < 8; ++i) fo.sig[fo.nsig++] = sig[i];
    for (; j < wait.size() && fo.nwait < 8; ++j) fo.wait[fo.nwait++] = wait[j];
    stress(st);
    prof_begin(st);
    if (int e = launch_flag_ops(fo, st)) return check_cuda(e, "flag ops");
    prof_end(st, 0.0, 0.0, 126 << 24);
  }
  return HP_OK;
}

void Engine::fork_streams() {
  if (forked_) return;
  cudaEvent_t e = pool_event();
  cudaEventRecord(e, stream_);
  cudaStreamWaitEvent(xs_, e, 0);
  for (int v = 0; v < N_; ++v) {
    if (vs_[v]) cudaStreamWaitEvent(vs_[v], e, 0);
    if (fs_[v]) cudaStreamWaitEvent(fs_[v], e, 0);
  }
  forked_ = true;
}


// The context stream waits for every side stream (all work issued so far is
// ordered before anything later on the context stream, e.g. a timing event).
hp_status Engine::join_exchange() {
  if (!dist_ || !forked_) return HP_OK;
  cudaEvent_t e = pool_event();
  cudaEventRecord(e, xs_);
  cudaStreamWaitEvent(stream_, e, 0);
  for (int v = 0; v < N_; ++v) {
    for (cudaStream_t sv : {vs_[v], fs_[v]}) {
      if (!sv) continue;
      cudaEvent_t ev = pool_event();
      cudaEventRecord(ev, sv);
      cudaStreamWaitEvent(stream_, ev, 0);
    }
  }
  for (auto& x : xacc_) std::fill(x.begin(), x.end(), nullptr);
  std::fill(xwl_.begin(), xwl_.end(), nullptr);
  std::fill(lastc_.begin(), lastc_.end(), nullptr);
  std::fill(lastw_.begin(), lastw_.end(), nullptr);
  forked_ = false;
  return check_cuda(cudaGetLastError(), "join");
}

hp_status Engine::ipc_handle(void* out) {
  if (sticky_) return sticky_;
  cudaIpcMemHandle_t h;
  if (int e = cudaIpcGetMemHandle(&h, arena_)) return check_cuda(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == kIpcBytes, "IPC handle size");
  memcpy(out, &h, kIpcBytes);
  return HP_OK;
}

hp_status Engine::connect(const void* handles, const void* comm_id) {
  if (sticky_) return sticky_;
  if (!dist_) return fail(HP_ERR_STATE, "hp_connect needs world > 1");
  if (connected_) return fail(HP_ERR_STATE, "already connected");
  if (cfg_.transport == HP_XPORT_NVLS)
    return fail(HP_ERR_STATE, "HP_XPORT_NVLS needs hp_connect_symmetric with a multicast mapping");
  for (int q = 0; q < G_; ++q) {
    if (q == rank_) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)q * kIpcBytes, kIpcBytes);
    void* p = nullptr;
    if (int e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess))
      return check_cuda(e, "cudaIpcOpenMemHandle");
    opened_.push_back(p);
    peer_[q] = (char*)p;
  }
  return finish_connect(comm_id);
}

hp_status Engine::connect_symmetric(const void* const* bases, void* mc, const void* comm_id) {
  if (sticky_) return sticky_;
  if (!dist_) return fail(HP_ERR_STATE, "hp_connect_symmetric needs world > 1");
  if (connected_) return fail(HP_ERR_STATE, "already connected");
  if (!ext_arena_) return fail(HP_ERR_STATE, "hp_connect_symmetric needs cfg.arena");
  if (cfg_.transport == HP_XPORT_NVLS && !mc)
    return fail(HP_ERR_STATE, "HP_XPORT_NVLS needs a multicast mapping");
  for (int q = 0; q < G_; ++q) {
    if (!bases[q] || ((uintptr_t)bases[q] & 255)) return fail(HP_ERR_INVALID, "bad peer base");
    if (q != rank_) peer_[q] = (char*)bases[q];
  }
  if ((const char*)bases[rank_] != (const char*)arena_)
    return fail(HP_ERR_INVALID, "peer_bases[rank] must be cfg.arena");
  mc_ = (char*)mc;
  return finish_connect(comm_id);
}

hp_status Engine::finish_connect(const void* comm_id) {
  if (const char* fb = getenv("HP_FLAG_BARRIER")) flag_barrier_ = atoi(fb) != 0;
  if (const char* pp = getenv("HP_P2P")) p2p_ = atoi(pp) != 0;
  if (const char* to = getenv("HP_FLAG_TIMEOUT_MS")) flag_timeout_ns_ = 1000000ull * strtoull(to, nullptr, 10);
  readers_.assign(G_, 0);
  if (comm_id) {
    std::string err;
    comm_ = comm_create(comm_id, G_, rank_, &err);
    if (!comm_) return fail(HP_ERR_COMM, err);
  } else {
    // co-located ranks (e.g. threads of one process sharing a GPU): no NCCL
    // communicator, so the barriers are the K7 device flags and the exchange
    // is the PEER path (NCCL refuses two ranks on one device)
    if (!flag_barrier_) return fail(HP_ERR_STATE, "connecting without a communicator needs the flag barrier");
    if (cfg_.transport == HP_XPORT_NCCL)
      return fail(HP_ERR_STATE, "HP_XPORT_NCCL needs a communicator id");
  }
  if (flag_barrier_) {
    if (int e = cudaMalloc((void**)&flag_err_, 8 * sizeof(int))) return check_cuda(e, "flag error");
    if (int e = cudaMemsetAsync(flag_err_, 0, 8 * sizeof(int), stream_))
      return check_cuda(e, "flag error");
  }
  // Stream priorities (HP_PRIO, default on): the exchange and the folds that
  // wait for it are the round's critical path; the accumulation of the next
  // wave has slack (the acc ring), so its CTAs yield to them.
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char* pr = getenv("HP_PRIO"))
    if (atoi(pr) == 0) prio_lo = prio_hi = 0;
  if (int e = cudaStreamCreateWithPriority(&xs_, cudaStreamNonBlocking, prio_hi))
    return check_cuda(e, "stream");
  // (the second exchange stream serves only the NVLS / peer split)
  if (cfg_.transport == HP_XPORT_NVLS)
    if (int e = cudaStreamCreateWithPriority(&xs2_, cudaStreamNonBlocking, prio_hi))
      return check_cuda(e, "stream");
  if (const char* ns = getenv("HP_NVLS_SPLIT")) nvls_split_ = std::max(0, std::min(100, atoi(ns)));
  xacc_.assign(N_, std::vector<cudaEvent_t>(R_, nullptr));
  xwl_.assign(N_, nullptr);
  lastc_.assign(N_, nullptr);
  lastw_.assign(N_, nullptr);
  vs_.assign(N_, nullptr);
  fs_.assign(N_, nullptr);
  // the most VW stages any GPU holds (1: C3 at 4 GPUs, C3 with two-stage VWs
  // at 8, one VW per GPU)
  int most = 0;
  for (int q = 0; q < G_; ++q) {
    int cnt = 0;
    for (int v = 0; v < N_; ++v) cnt += lay_[q].has[v] ? 1 : 0;
    most = std::max(most, cnt);
  }
  const bool one_stage_sgd = cfg_.transport == HP_XPORT_PEER && cfg_.momentum == 0.f && most <= 1;
  // Split acc / fold launches by default (row a9) where they measured faster:
  // one VW stage per GPU, SGD, peer exchange, one process per GPU (a
  // communicator), and at least 16 hardware work queues
  // (CUDA_DEVICE_MAX_CONNECTIONS, read by the CUDA runtime at context
  // creation; with the default 8 the fold stream shares a queue with the
  // exchange or accumulation stream and the split launches serialise behind
  // it). C3 at 4 GPUs: 1.074 -> 1.012-1.016 ms per round with the
  // accumulation grid at 2.5 CTAs per SM (profiles/r02/c3_overlap_g4/).
  bool auto_split = false;
  if (const char* sf = getenv("HP_SPLIT_FOLDS")) {
    split_folds_ = atoi(sf) != 0;
  } else {
    const char* mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    auto_split = one_stage_sgd && comm_ && !convex_ && mc && atoi(mc) >= 16;
    split_folds_ = auto_split;
  }
  if (const char* pp = getenv("HP_PULL_PUSH")) push_pull_ = atoi(pp) != 0;
  for (int v = 0; v < N_; ++v)
    if (vw_[v].here)
    {
      if (int e = cudaStreamCreateWithPriority(&vs_[v], cudaStreamNonBlocking, prio_lo))
        return check_cuda(e, "stream");
      if (split_folds_)                 // fold streams only for split acc / fold launches
        if (int e = cudaStreamCreateWithPriority(&fs_[v], cudaStreamNonBlocking, prio_hi))
          return check_cuda(e, "stream");
    }
  if (const char* xb = getenv("HP_XBLOCKS")) {
    xblocks_ = atoi(xb);
  } else if (one_stage_sgd) {
    // one VW stage per GPU, SGD (C3 at 4 GPUs, C3 with two-stage VWs at 8):
    // the owners' apply launches on 128 CTAs measured 5% faster per round
    // (1.09 vs 1.15 ms, profiles/r02/multi_g4_knobs/); with several stages per
    // GPU (C3 at 2 GPUs) or heavy-ball momentum (C5) the bound cost 10-15%
    xblocks_ = 128;
  }
  if (const char* ab = getenv("HP_ABLOCKS")) {
    ablocks_ = atoi(ab);
  } else if (auto_split) {
    // the split accumulation launches on 2.5 CTAs per SM leave room beside
    // them for the exchange launch's CTAs (2 per SM: 1.033 ms, 3: 1.10,
    // full grid: 1.15; profiles/r02/c3_overlap_g4/)
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ablocks_ = sms > 0 ? sms * 5 / 2 : 0;
  }
  // HP_AGRID=1: accumulation launches non-persistent (CTAs retire every U
  // chunks), so the high-priority exchange stream's launches start promptly
  if (const char* ag = getenv("HP_AGRID"))
    if (atoi(ag) == 1) ablocks_ = -1;
  // everyone's init writes are complete before anyone reads a peer (without a
  // communicator: the first flag barrier, epoch 1 on every rank -- the flag
  // arrays were zeroed by every rank's hp_init_ex, which the caller ordered
  // before any hp_connect_symmetric)
  if (comm_) {
    if (comm_->barrier(stream_) != 0) return fail(HP_ERR_COMM, comm_->error());
  } else {
    ++epoch_;
    FlagBarrier fb;
    memset(&fb, 0, sizeof fb);
    fb.G = G_;
    fb.me = rank_;
    fb.epoch = epoch_;
    fb.err = flag_err_;
    fb.timeout_ns = flag_timeout_ns_;
    for (int q = 0; q < G_; ++q) fb.flags[q] = (unsigned long long*)(peer_[q] + lay_[q].flag_off);
    if (int e = launch_flag_barrier(fb, stream_)) return check_cuda(e, "flag barrier");
  }
  connected_ = true;
  if (hp_status st = check_cuda(cudaStreamSynchronize(stream_), "connect sync")) return st;
  if (flag_err_) {
    int bad = 0;
    if (int e = cudaMemcpyAsync(&bad, flag_err_, sizeof bad, cudaMemcpyDeviceToHost, stream_))
      return check_cuda(e, "flag error");
    if (int e = cudaStreamSynchronize(stream_)) return check_cuda(e, "flag error");
    if (bad) {
      sticky_ = HP_ERR_COMM;
      return fail(HP_ERR_COMM, "connect: a rank did not reach the first flag barrier");
    }
  }
  return HP_OK;
}

}  // namespace hp

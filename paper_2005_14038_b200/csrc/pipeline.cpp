// pipeline.cpp -- intra-VW pipeline schedule (section 4, P:760-806;
// SURVEY.md 8(f) NEXT-1): the min-max layer partitioner under the
// stage-dependent memory requirement and the pipeline simulator under
// scheduling conditions 1-3. Host C++, exported through include/hetpipe.h
// (hp_partition, hp_pipeline_simulate, hp_pipeline_tau_latency, hp_max_m).
// Independent of oracle/pipeline.py (brute force / plain event loop).
//
// Times are integer nanoseconds; every rounding is round-half-even of one
// double expression, so results are reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <queue>
#include <vector>

#include "../../include/hetpipe.h"

namespace {

constexpr int64_t kInf = std::numeric_limits<int64_t>::max() / 4;
constexpr int64_t kParamOverhead = 3;   // weights + gradients + optimizer state

int64_t rnd(double x) { return (int64_t)std::nearbyint(x); }

// Stage costs of one GPU order: prefix sums make every (stage, lo, hi) O(1).
struct Coster {
  const hp_unit* u;
  int L, k, Nm, batch;
  std::vector<hp_gpu> g;                 // stage order
  double intra, inter;
  std::vector<int64_t> pf, pp, pr;       // prefix fwd_flops, params, resident

  void init() {
    pf.assign(L + 1, 0);
    pp.assign(L + 1, 0);
    pr.assign(L + 1, 0);
    for (int i = 0; i < L; ++i) {
      pf[i + 1] = pf[i] + u[i].fwd_flops;
      pp[i + 1] = pp[i] + u[i].params;
      pr[i + 1] = pr[i] + u[i].act_resident;
    }
  }
  double bw(int a, int b) const { return g[a].node == g[b].node ? intra : inter; }
  int64_t depth(int q) const { return std::min<int64_t>(Nm, 2 * (k - 1 - q) + 1); }
  bool fits(int q, int lo, int hi) const {
    const int64_t need = kParamOverhead * 4 * (pp[hi] - pp[lo]) + depth(q) * 4 * batch * (pr[hi] - pr[lo]);
    return (double)need <= g[q].mem_bytes;
  }
  int64_t fwd(int q, int lo, int hi) const {
    return rnd((double)((pf[hi] - pf[lo]) * batch) / g[q].flops_per_s * 1e9);
  }
  int64_t comm(int cut, double b) const {   // activation leaving unit cut-1
    return rnd((double)(u[cut - 1].act_out * 4 * batch) / b * 1e9);
  }
  void costs(int q, int lo, int hi, int64_t out[4]) const {
    out[0] = fwd(q, lo, hi);
    out[1] = 2 * out[0];
    out[2] = q > 0 ? comm(lo, bw(q - 1, q)) : 0;
    out[3] = q < k - 1 ? comm(hi, bw(q, q + 1)) : 0;
  }
  int64_t time(int q, int lo, int hi) const {
    if (!fits(q, lo, hi)) return kInf;
    int64_t c[4];
    costs(q, lo, hi, c);
    return c[0] + c[1] + c[2] + c[3];
  }
};

// Min-max split of one order: suffix DP, then the lexicographically smallest
// cuts that achieve the optimum. Returns kInf if nothing fits.
int64_t best_split(const Coster& C, std::vector<int>* cuts) {
  const int L = C.L, k = C.k;
  // suf[q][lo]: best bottleneck of stages q..k-1 over units lo..L-1
  std::vector<std::vector<int64_t>> suf(k + 1, std::vector<int64_t>(L + 1, kInf));
  suf[k][L] = 0;
  for (int q = k - 1; q >= 0; --q)
    for (int lo = 0; lo < L; ++lo) {
      int64_t b = kInf;
      for (int hi = lo + 1; hi <= L; ++hi) {
        if (suf[q + 1][hi] >= kInf) continue;
        const int64_t t = C.time(q, lo, hi);
        if (t >= kInf) continue;
        b = std::min(b, std::max(t, suf[q + 1][hi]));
      }
      suf[q][lo] = b;
    }
  const int64_t B = suf[0][0];
  if (B >= kInf) return kInf;
  cuts->assign(1, 0);
  int lo = 0;
  for (int q = 0; q < k; ++q) {
    for (int hi = lo + 1; hi <= L; ++hi) {
      if (suf[q + 1][hi] >= kInf) continue;
      const int64_t t = C.time(q, lo, hi);
      if (t < kInf && std::max(t, suf[q + 1][hi]) <= B) {
        cuts->push_back(hi);
        lo = hi;
        break;
      }
    }
  }
  return B;
}

// The pipeline of one VW (conditions 1-3 of P:796-803). Task kinds: 0 = F,
// 1 = B, 2 = FB (the last partition's fused forward+backward).
struct Sim {
  int k, Nm;
  int64_t P;
  const int64_t* c;   // k x 4: fwd, bwd, comm_in_fwd, comm_in_bwd
  struct Task {
    int64_t ready;
    int kind;
    int64_t p;
  };
  std::vector<std::vector<Task>> q;       // per GPU: tasks whose inputs arrived
  std::vector<int64_t> free_at;
  std::vector<std::vector<int64_t>> last; // per GPU, per kind: last minibatch done
  std::vector<int64_t> start, comp;
  int64_t ncomp = 0;

  void admit(int64_t p, int64_t t) {
    start[p] = t;
    q[0].push_back({t, k == 1 ? 2 : 0, p});
  }
  bool eligible(int g, const Task& t) const { return last[g][t.kind] == t.p - 1; }

  void run() {
    q.assign(k, {});
    free_at.assign(k, 0);
    last.assign(k, std::vector<int64_t>(3, 0));
    start.assign(P + 1, 0);
    comp.assign(P + 1, 0);
    for (int64_t p = 1; p <= std::min<int64_t>(Nm, P); ++p) admit(p, 0);
    while (ncomp < P) {
      int bg = -1;
      int64_t bs = 0;
      size_t bi = 0;
      for (int g = 0; g < k; ++g) {
        int64_t mr = kInf;
        for (const Task& t : q[g])
          if (eligible(g, t)) mr = std::min(mr, t.ready);
        if (mr >= kInf) continue;
        const int64_t s = std::max(free_at[g], mr);
        // FIFO among tasks ready by s: earliest ready, backward first, lower p
        size_t pick = q[g].size();
        for (size_t i = 0; i < q[g].size(); ++i) {
          const Task& t = q[g][i];
          if (!eligible(g, t) || t.ready > s) continue;
          if (pick == q[g].size()) {
            pick = i;
            continue;
          }
          const Task& b = q[g][pick];
          const int tk = t.kind == 0 ? 1 : 0, bk = b.kind == 0 ? 1 : 0;
          if (t.ready < b.ready || (t.ready == b.ready && (tk < bk || (tk == bk && t.p < b.p))))
            pick = i;
        }
        if (bg < 0 || s < bs) {
          bg = g;
          bs = s;
          bi = pick;
        }
      }
      const Task t = q[bg][bi];
      q[bg].erase(q[bg].begin() + (long)bi);
      const int64_t* cg = c + 4 * bg;
      const int64_t dur = t.kind == 0 ? cg[0] : t.kind == 1 ? cg[1] : cg[0] + cg[1];
      const int64_t end = bs + dur;
      free_at[bg] = end;
      last[bg][t.kind] = t.p;
      if (t.kind == 0) {
        const int nx = bg + 1;
        q[nx].push_back({end + c[4 * nx + 2], nx == k - 1 ? 2 : 0, t.p});
      } else if (bg > 0) {
        q[bg - 1].push_back({end + c[4 * (bg - 1) + 3], 1, t.p});
      } else {
        comp[t.p] = end;
        ++ncomp;
        if (t.p + Nm <= P) admit(t.p + Nm, end);   // START(p+Nm) at COMPLETE(p)
      }
    }
  }
};

bool valid_costs(const int64_t* c, int k) {
  for (int i = 0; i < 4 * k; ++i)
    if (c[i] < 0) return false;
  for (int g = 0; g < k; ++g)
    if (c[4 * g] + c[4 * g + 1] <= 0) return false;
  return true;
}

}  // namespace

extern "C" {

hp_status hp_partition(const hp_unit* units, int32_t L, const hp_gpu* gpus, int32_t k,
                       int32_t Nm, int32_t batch, double intra_bps, double inter_bps,
                       int32_t* order_out, int32_t* cuts_out, int64_t* stage_costs_out,
                       int64_t* bottleneck_ns) {
  if (!units || !gpus || L < 1 || k < 1 || k > 8 || k > L || Nm < 1 || batch < 1 ||
      !(intra_bps > 0) || !(inter_bps > 0))
    return HP_ERR_INVALID;
  for (int i = 0; i < k; ++i)
    if (!(gpus[i].flops_per_s > 0)) return HP_ERR_INVALID;
  std::vector<int> perm(k);
  for (int i = 0; i < k; ++i) perm[i] = i;
  int64_t best = kInf;
  std::vector<int> best_perm, best_cuts;
  Coster C{units, L, k, Nm, batch, {}, intra_bps, inter_bps, {}, {}, {}};
  C.init();
  do {   // permutations in lexicographic order: the first optimum wins ties
    C.g.clear();
    for (int i = 0; i < k; ++i) C.g.push_back(gpus[perm[i]]);
    std::vector<int> cuts;
    const int64_t b = best_split(C, &cuts);
    if (b < best) {
      best = b;
      best_perm = perm;
      best_cuts = cuts;
    }
  } while (std::next_permutation(perm.begin(), perm.end()));
  if (best >= kInf) return HP_WOULD_BLOCK;   // no feasible partition (memory)
  C.g.clear();
  for (int i = 0; i < k; ++i) C.g.push_back(gpus[best_perm[i]]);
  for (int i = 0; i < k; ++i) {
    if (order_out) order_out[i] = best_perm[i];
    if (stage_costs_out) C.costs(i, best_cuts[i], best_cuts[i + 1], stage_costs_out + 4 * i);
  }
  if (cuts_out)
    for (int i = 0; i <= k; ++i) cuts_out[i] = best_cuts[i];
  if (bottleneck_ns) *bottleneck_ns = best;
  return HP_OK;
}

int32_t hp_max_m(const hp_unit* units, int32_t L, const hp_gpu* gpus, int32_t k, int32_t batch,
                 double intra_bps, double inter_bps) {
  for (int32_t nm = 2 * k - 1; nm >= 1; --nm)
    if (hp_partition(units, L, gpus, k, nm, batch, intra_bps, inter_bps, nullptr, nullptr,
                     nullptr, nullptr) == HP_OK)
      return nm;
  return 0;
}

hp_status hp_pipeline_simulate(const int64_t* stage_costs, int32_t k, int32_t Nm, int64_t P,
                               int64_t* start_out, int64_t* complete_out) {
  if (!stage_costs || k < 1 || k > 64 || Nm < 1 || P < 1 || !valid_costs(stage_costs, k))
    return HP_ERR_INVALID;
  try {
    Sim s{k, Nm, P, stage_costs, {}, {}, {}, {}, {}, 0};
    s.run();
    for (int64_t p = 1; p <= P; ++p) {
      if (start_out) start_out[p - 1] = s.start[p];
      if (complete_out) complete_out[p - 1] = s.comp[p];
    }
  } catch (...) {
    return HP_ERR_OOM;
  }
  return HP_OK;
}

hp_status hp_pipeline_tau_latency(const int64_t* stage_costs, int32_t k, int32_t Nm, int64_t P,
                                  int64_t* tau_ns, int64_t* latency_ns) {
  if (P <= 0) P = 24 * (int64_t)std::max(Nm, 1);
  if (P < 4) return HP_ERR_INVALID;
  std::vector<int64_t> comp(P);
  if (hp_status st = hp_pipeline_simulate(stage_costs, k, Nm, P, nullptr, comp.data())) return st;
  const int64_t a = P / 4, b = 3 * P / 4;      // middle half: fill and drain excluded
  if (tau_ns) *tau_ns = (comp[b - 1] - comp[a - 1]) / (b - a);
  if (latency_ns) *latency_ns = comp[0];
  return HP_OK;
}

}  // extern "C"

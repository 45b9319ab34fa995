// tick_desc.h -- the fused per-tick device program (internal to libhetpipe).
//
// Every WSP operation is element-wise in the parameter index (PAPER.md P:839
// w_local += u_p, P:922 wave aggregate, P:929 w_global += u~, P:949 pull), so all
// operations of one controller tick can run in ONE pass over the parameters with
// every intermediate held in registers. The host engine builds a TickDesc per
// tick in the paper's phase order (Z5):
//   1. completes  u_j = fl(-lr*g(v_j,p_j));  a_j = first ? u_j : acc_j + u_j
//   2. applies    in commit order: w_global += a (or m = mu*m + a; w += m)
//   3. groups     per VW: w = pull ? w_global (+ partial u~) : w_local;
//                 then the VW's due folds w += u_f in minibatch order; store w
// Passed by value as a __grid_constant__ kernel parameter (< 4 KB).
#pragma once
#include <stdint.h>

namespace hp {

constexpr int kMaxC = 8;    // completes per tick (at most one per VW)
constexpr int kMaxA = 8;    // applies per launch
constexpr int kMaxG = 8;    // w_local groups per launch (one per VW)
constexpr int kMaxF = 48;   // folds per launch

enum : uint32_t { kFirst = 1u, kStoreAcc = 2u, kLoadAcc = 4u };

struct DComplete {
  float* acc;          // acc slot of the wave p belongs to
  const float* grad;   // EXTERNAL gradient (local shard) or nullptr
  uint32_t v, p;
  uint32_t flags;      // kFirst | kStoreAcc
  uint32_t pad;
};

struct DApply {
  const float* src;    // acc slot in memory, used when reg < 0
  int32_t reg;         // complete index whose register holds u~, or -1
  int32_t pad;
};

struct DFold {
  const float* grad;   // EXTERNAL gradient or nullptr
  uint32_t v, p;
  int32_t reg;         // complete index whose register holds u_p, or -1
  int32_t pad;
};

struct DGroup {
  float* wl;             // w_local of this VW (local shard)
  const float* partial;  // AT_LEAST pull: open-wave acc in memory, or nullptr
  int32_t pull;          // 1: base = w_global (+partial); 0: base = w_local
  int32_t partial_reg;   // complete index holding the partial, or -1
  int32_t f_begin, f_end;
};

struct TickDesc {
  int64_t n;            // params in this rank's shard
  int64_t blk_base;     // param_begin / 4 (param_begin is a multiple of 32)
  float* wg;            // w_global shard
  float* m;             // momentum shard (nullptr for SGD)
  float neg_lr;         // -lr (negation is exact, Z10)
  float mu;             // momentum
  uint32_t key0, key1;  // Philox key = seed
  int32_t nc, na, ng, nf;
  int32_t wg_load;      // w_global must be read (applies or pulls present)
  int32_t pad;
  DComplete c[kMaxC];
  DApply a[kMaxA];
  DGroup g[kMaxG];
  DFold f[kMaxF];
};

static_assert(sizeof(TickDesc) <= 4000, "TickDesc must fit a kernel parameter");

// Launch the fused tick kernel (kernels.cu). grad_mode: HP_GRAD_*.
// Returns a cudaError_t as int.
int launch_tick(const TickDesc& d, int grad_mode, bool momentum, void* stream);
// out[i] = w0(param_begin + i) over the shard (kernels.cu, reading Z8).
int launch_init(float* out, int64_t n, int64_t param_begin, int w0_mode, int grad_mode,
                uint32_t key0, uint32_t key1, void* stream);

}  // namespace hp

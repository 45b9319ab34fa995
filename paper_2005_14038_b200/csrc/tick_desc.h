// tick_desc.h -- the fused per-tick device program (internal to libhetpipe).
//
// Every WSP operation is element-wise in the parameter index (PAPER.md P:839
// w_local += u_p, P:922 wave aggregate, P:929 w_global += u~, P:949 pull), so all
// operations of one controller tick run in ONE pass over the parameters. The
// host engine builds a TickDesc per tick; the kernel executes, per param:
//   A. memory applies  w_global += u~ (or m = mu*m + u~; w += m) for pushes whose
//                      u~ is in an acc slot, in commit order (Z4, Z11)
//   B. completes       u = fl(-lr*g(v,p)); a = first ? u : acc + u;
//                      [store acc]; [apply a now: this tick's pushes, which come
//                      last in commit order]; [inline fold w_local += u]
//   C. store w_global (and m) if anything was applied
//   D. w_local groups  w = pull ? w_global (+ partial u~, AT_LEAST) : w_local;
//                      then the VW's due folds w += u in minibatch order; store
// Passed by value as a __grid_constant__ kernel parameter (< 4 KB).
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace hp {

constexpr int kMaxC = 8;    // completes per launch (at most one per VW per tick)
constexpr int kMaxA = 16;   // memory-sourced applies per launch
constexpr int kMaxG = 8;    // w_local groups per launch (one per VW)
constexpr int kMaxF = 40;   // folds per launch
constexpr int kMaxS = 32;   // source segments per launch
constexpr int kMaxP = 16;   // pushed-pull store targets per launch
constexpr int kTileSlots = 64;   // launch streams with dynamic tile counters per context
constexpr size_t kTickBatch = 512;   // tick descriptors per multi-tick launch (captures)

enum : uint32_t {
  kFirst = 1u,       // first minibatch of its wave: a = u
  kStoreAcc = 2u,    // write a back to the acc slot
  kLoadAcc = 4u,     // read the acc slot (not first)
  kApplyNow = 8u,    // w_global += a right after this complete (commit order)
  kFoldInline = 16u, // w_local(v) += u right here (the VW's only due fold)
  kStashAfter = 32u, // CONVEX: START(p+Nm) reads the folded w_local -> stash slot
  kSnapAcc = 64u     // F > 1: copy the loaded acc (before this u) to `snap`
};

struct DComplete {
  float* acc;          // acc slot of the wave p belongs to
  const float* grad;   // EXTERNAL gradient (local shard) or nullptr
  float* wl;           // w_local for kFoldInline, else nullptr
  float* stash;        // CONVEX: slot (p-1) mod Nm holding w_p (kStashAfter rewrites it)
  float* snap;         // kSnapAcc: the waiting VW's open-clock aggregate (reading Z25)
  uint32_t v, p;
  uint32_t flags;
  float neg_lr;        // -eta of u_p: -lr, or -sigma/sqrt(t) (hp_config.lr_schedule)
};

// A source array split into segments by local index: element i of the launch
// reads seg.ptr[i] for the first segment with i < seg.end (ptr pre-offset so the
// launch's local index addresses it; may point into a peer GPU's memory).
struct DSeg {
  const float* ptr;
  int64_t end;
};

// Pull by the shard owner (distributed placements): after phase C the final
// w_global of local index i in [lo, hi) is also stored at ptr[i], a pulled
// VW's w_local slice that may live on a peer GPU (NVLink stores).
struct DStore {
  float* ptr;
  int64_t lo, hi;
};

struct DApply {
  int32_t seg_begin, seg_end;   // acc slice(s) holding u~ of an earlier push
};

// One op of a w_local group, in order: FOLD w += u_p (u regenerated, or from
// `grad`; CONVEX reads w_p from `stash`), or STASH (CONVEX: a START reads w
// now: stash <- w).
struct DFold {
  const float* grad;   // EXTERNAL gradient or nullptr (synthetic: regenerate)
  float* stash;        // CONVEX: FOLD reads w_p here; STASH writes w here
  uint32_t v, p;
  uint32_t op;         // 0 FOLD, 1 STASH
  float neg_lr;        // -eta of u_p (as DComplete::neg_lr)
};

struct DGroup {
  float* wl;             // w_local of this VW (local shard)
  const float* partial;  // AT_LEAST pull: open-wave acc slot, or nullptr
  int32_t pull;          // 0: base = w_local; 1: base = this launch's w_global
                         // (+partial); 2: base = w_global read through segments
  int32_t f_begin, f_end;
  int32_t seg_begin, seg_end;
  int32_t pad;
};

struct TickDesc {
  int64_t n;            // params in this rank's shard
  int64_t blk_base;     // param_begin / 4 (param_begin is a multiple of 32)
  float* wg;            // w_global shard
  float* m;             // momentum shard (nullptr for SGD)
  float neg_lr;         // -lr (unused by the kernels: every op carries its own -eta)
  float mu;             // momentum
  float conv_a, conv_sigma;   // CONVEX workload
  uint32_t key0, key1;  // Philox key = seed
  int32_t nc, na, ng, nf;
  int32_t wg_load;      // w_global must be read (applies or pulls present)
  int32_t wg_store;     // w_global (and m) must be written (applies present)
  DComplete c[kMaxC];
  DApply a[kMaxA];
  DGroup g[kMaxG];
  DFold f[kMaxF];
  DSeg s[kMaxS];
  int32_t ns;
  int32_t wgs_begin, wgs_end;   // if non-empty: w_global registers are loaded from
                                // these segments (remote shards) instead of wg
  int32_t np;                   // store targets of the owner-side pull
  int32_t pf;                   // L2 prefetch distance in chunk rounds (0 = off;
                                // only when every load of the launch is local)
  int32_t lean;                 // completes only (no applies / w_global / groups /
                                // pull stores): the phase-B-only kernel instance
  unsigned long long* ctr;      // dynamic tile scheduling (nullptr = static grid
  unsigned int* done;           // stride): tile counter and finished-CTA count of
                                // the launch stream, both 0 between launches
  DStore pd[kMaxP];
};

static_assert(sizeof(TickDesc) <= 4096, "TickDesc must fit a kernel parameter");

// A TickDesc in device memory (multi-tick batches): 16-byte aligned stride, so
// the kernel stages it with one 16-byte load per thread.
struct alignas(16) TickDescPad {
  TickDesc d;
};

// Buffer passes of one launch (each = 4 bytes per param): the algorithmic
// bytes the fused tick must move, used for the roofline.
inline int tick_streams(const TickDesc& d) {
  int s = d.wg_load + (d.wg_store ? 1 : 0);   // (+ the owner-side pull stores: emit())
  if (d.m && d.wg_store) s += 2;
  s += d.na;
  for (int j = 0; j < d.nc; ++j) {
    const uint32_t f = d.c[j].flags;
    s += ((f & kLoadAcc) ? 1 : 0) + ((f & kStoreAcc) ? 1 : 0) + (d.c[j].grad ? 1 : 0) +
         ((f & kFoldInline) ? 2 : 0) + (d.c[j].stash ? 1 : 0) + ((f & kStashAfter) ? 1 : 0) +
         ((f & kSnapAcc) ? 1 : 0);
  }
  for (int g = 0; g < d.ng; ++g) {
    s += 1 + (d.g[g].pull == 1 ? 0 : 1) + (d.g[g].partial ? 1 : 0);
    for (int k = d.g[g].f_begin; k < d.g[g].f_end; ++k)
      s += (d.f[k].grad ? 1 : 0) + (d.f[k].stash ? 1 : 0);
  }
  return s;
}

// The synchronisation share of tick_streams(): w_global load/store, momentum,
// memory-sourced applies (the u~ reads of a4/a5) and the pull writes of w_local
// (a7, plus the AT_LEAST partial). The rest is accumulation (a2/a3).
inline int tick_sync_streams(const TickDesc& d) {
  int s = d.wg_load + (d.wg_store ? 1 : 0);
  if (d.m && d.wg_store) s += 2;
  s += d.na;
  for (int g = 0; g < d.ng; ++g)
    if (d.g[g].pull) s += 1 + (d.g[g].pull == 2 ? 1 : 0) + (d.g[g].partial ? 1 : 0);
  return s;
}

// Lockstep exchange through the NVSwitch (HP_XPORT_NVLS, include/hetpipe.h):
// over this rank's PS shard, u = multimem.ld_reduce(mc_acc) (the sum of every
// GPU's pushed u~ at that index), w_global += u, and if mc_wl is set
// multimem.st(mc_wl, w_global) writes the pulled value into every GPU's
// w_local. src/dst are the same buffers through unicast peer mappings (used
// only by the host emulation in tests/emu; the device kernel uses mc_*).
struct NvlsDesc {
  int64_t n;             // params of this rank's PS shard
  float* wg;             // w_global shard
  const float* mc_acc;   // multicast address of the acc slot at the shard's first param
  float* mc_wl;          // multicast address of w_local at the shard's first param, or nullptr
  int32_t G;
  int32_t pad;
  unsigned long long* ctr;   // dynamic tiles (nullptr = static grid stride), as TickDesc
  unsigned int* done;
  const float* src[8];   // per rank: acc slot at the shard's first param (unicast)
  float* dst[8];         // per rank: w_local at the shard's first param (unicast)
};
int launch_nvls(const NvlsDesc& d, void* stream, int max_blocks = 0);

// K7 readiness barrier among G ranks (engine.cpp xbarrier): flags[q] is rank
// q's flag array (one uint64 per source rank), mapped into this process.
struct FlagBarrier {
  unsigned long long* flags[8];
  int* err;                    // device int set to 1 if a wait timed out
  unsigned long long epoch;
  unsigned long long timeout_ns;   // wait deadline (HP_FLAG_TIMEOUT_MS, default 10 s)
  int32_t G, me;
};
int launch_flag_barrier(const FlagBarrier& fb, void* stream);

// Point-to-point readiness flags (engine_dist.cpp): one
// tiny kernel that publishes `val` into up to 8 flag words (after a system
// fence: everything earlier on the stream is visible to whoever sees a flag)
// and waits until up to 8 flag words hold >= `val`. Flags are monotonic
// epochs, so a later signal satisfies an earlier wait.
struct FlagOps {
  unsigned long long* sig[8];
  const unsigned long long* wait[8];
  unsigned long long val;
  unsigned long long timeout_ns;   // wait deadline (HP_FLAG_TIMEOUT_MS, default 10 s)
  int* err;                    // device int set to 1 if a wait timed out
  int32_t nsig, nwait;
};
int launch_flag_ops(const FlagOps& fo, void* stream);
// Run `count` tick descriptors (device memory, in order) in one launch over
// [0, n) of a single-rank context (static element -> thread map; FLOAT,
// DYADIC, CONVEX). Returns a cudaError_t as int.
int launch_multi_tick(const TickDescPad* descs, int count, int64_t n, int grad_mode, bool momentum,
                      void* stream);
// Load every kernel instance now (once per device; lazy module loading could
// otherwise stall a spinning flag barrier). Returns a cudaError_t as int.
int preload_kernels();
// hp_launch_floor: an empty one-CTA kernel launched with the PDL attribute.
int launch_empty(void* stream);
// HP_STRESS: an idle one-warp kernel of `ns` nanoseconds on `stream`.
int launch_spin(unsigned long long ns, void* stream);

// Launch the fused tick kernel (kernels.cu). grad_mode: HP_GRAD_*.
// Returns a cudaError_t as int.
// max_blocks > 0 bounds the grid (exchange launches that share the GPU with
// accumulation launches on other streams); 0 = default grid.
int launch_tick(const TickDesc& d, int grad_mode, bool momentum, void* stream,
                int max_blocks = 0);
// out[i] = w0(param_begin + i) over the shard (kernels.cu, reading Z8).
int launch_init(float* out, int64_t n, int64_t param_begin, int w0_mode, int grad_mode,
                uint32_t key0, uint32_t key1, void* stream);

}  // namespace hp

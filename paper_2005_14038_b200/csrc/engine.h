// engine.h -- WSP protocol engine of libhetpipe: host-side clocks, gate,
// commit log and version trace, plus the per-tick batch that becomes one fused
// kernel launch (tick_desc.h). Independent of oracle/ (shares no code).
//
// Paper mapping (P:n = PAPER.md line n):
//   complete()  COMPLETE(v,p): u_p into the open wave's acc slot and a
//               pending fold w_local += u_p, materialised before the
//               next START that reads w_local (JIT fold, reading Z3).
//   push()      PUSH(v,c): commit log append, c_local = c+1, c_global = min
//               (P:917-930). The PS apply is deferred to the first observer
//               (a pull or a read) unless apply_mode = ON_ARRIVAL (reading Z4).
//   admit()     GATE/PULL(v) for the gated START (c+2)*Nm (Z7, Z17).
//   tick_end()  START phase records + one fused launch (Z5).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/hetpipe.h"
#include "comm.h"
#include "tick_desc.h"

namespace hp {

// Where a rank's buffers live in its arena (same function on every rank, so
// any rank can address any peer's buffers through the peer's arena base).
struct RankLayout {
  int64_t s0 = 0, s1 = 0;             // PS shard [s0, s1) (global params)
  size_t wg_off = 0, m_off = 0, x_off = 0, bytes = 0;   // x: NCCL staging (shard)
  size_t flag_off = 0;                // K7 readiness flags: uint64 per source rank
  std::vector<int64_t> a, len;        // per VW: local stage [a, a+len)
  std::vector<char> has;              // per VW: a stage lives on this rank
  std::vector<size_t> wl_off;
  std::vector<std::vector<size_t>> acc_off;
  std::vector<std::vector<size_t>> stash_off;   // CONVEX
  std::vector<size_t> snap_off;                 // F > 1, STRICT
};

struct VW {
  int64_t started = 0, completed = 0, c_local = 0;
  int64_t a = 0;                 // own-update cursor a_v (logical)
  int64_t held_g = 0, held_K = 0;
  bool at_gate = false, blocked = false;
  int64_t t_block = 0, wait = 0, pulls = 0;
  bool waited_last = false;      // its latest admission followed a BLOCK
  int64_t acc_count = 0;         // completions in the open wave
  std::vector<int64_t> backlog;  // completions while waiting at the gate (Z17)
  // Ops on w_local not yet on the device, in order: p > 0 = FOLD u_p; p < 0 =
  // STASH (CONVEX: START(-p) reads w_local now, into stash slot (-p-1) mod Nm)
  std::vector<int64_t> pending_folds;
  int64_t a0 = 0, len = 0;       // this rank's stage of the VW (global range)
  bool here = false;             // the VW has a stage (possibly empty) on this rank
  float* wl = nullptr;
  std::vector<float*> acc;       // ring of R slots; wave c -> slot c % R
  std::vector<float*> stash;     // CONVEX: ring of Nm slots; w_p -> slot (p-1) % Nm
  float* snap = nullptr;         // F > 1, STRICT: acc of the open clock when the VW
  bool snap_valid = false;       //   reached its gate, if the backlog joined acc since
  const float* pull_partial = nullptr;  // pull base = w_global + this (or nullptr)
  std::vector<const float*> grad_of_slot;  // EXTERNAL: grad of minibatch p in slot (p-1)%Nm
  std::vector<float*> grad_ring;           // library-owned copies of host gradients
};

class Engine {
 public:
  explicit Engine(const hp_config& cfg);
  ~Engine();
  hp_status init();

  hp_status complete(int v, int64_t p, const float* grad_dev, const float* grad_host,
                     bool* wave_end);
  hp_status push(int v, int64_t c);
  hp_status clock(int v, int64_t* c_local, int64_t* c_global);
  hp_status admit(int v, std::vector<int64_t>* started);
  hp_status tick_end(std::vector<std::pair<int, int64_t>>* ungated);
  hp_status flush_applies();
  hp_status ipc_handle(void* out);
  hp_status connect(const void* handles, const void* comm_id);
  hp_status connect_symmetric(const void* const* bases, void* mc, const void* comm_id);
  int64_t arena_bytes() const { return (int64_t)layout_of(rank_).bytes; }
  void plan_layout();
  bool distributed() const { return dist_; }
  int64_t local_len(int which) const;
  double nvl_bytes() const { return nvl_bytes_; }
  // launch every queued op (side streams keep running)
  hp_status flush_queued() {
    if (!(bc_.empty() && ba_.empty() && bpull_.empty() && !has_due_folds()))
      if (hp_status st = flush()) return st;
    return HP_OK;
  }
  // ... and order all of it before later work on the context stream
  hp_status flush_pending() {
    if (hp_status st = flush_queued()) return st;
    return join_exchange();
  }
  hp_status sync();
  hp_status drain();                  // launched work done (deferred applies stay deferred)
  hp_status check_flag_err();         // HP_ERR_COMM if a K7 flag wait timed out
  hp_status read(int which, int64_t off, int64_t cnt, float* dst);
  // CUDA-graph capture of the device work of a controller advance
  // (hp_schedule_capture): begin -> the caller advances -> end(graph exec)
  hp_status capture_begin();
  hp_status capture_end(bool ok, cudaGraphExec_t* exec);
  hp_status graph_launch(cudaGraphExec_t exec);
  bool graph_pending() const { return graph_pending_; }
  void* stream() const { return stream_; }
  hp_status launch_floor(int n, bool graph, float* us);

  void set_tick(int64_t t) { tick_ = t; }
  bool at_gate(int v) const { return vw_[v].at_gate; }
  bool done() const;
  int64_t commits() const { return (int64_t)commit_.size(); }
  const hp_config& cfg() const { return cfg_; }
  int64_t last_p() const { return last_p_; }
  hp_status fail(hp_status s, const std::string& msg);
  hp_status sticky() const { return sticky_; }
  const std::string& error() const { return err_; }
  std::string& trace() { return trace_; }
  void set_trace(bool on) { trace_on_ = on; }
  void stats(hp_stats* out) const;
  hp_status profile_enable(bool on);
  hp_status profile_read(double* ms, double* bytes, int64_t* launches);
  hp_status profile_sync(int64_t max, float* ms, int32_t* vw, int32_t* waited, int64_t* n);
  hp_status profile_launches(int64_t max, float* ms, double* bytes, int32_t* shape,
                             double* sync_bytes, float* start_ms, int64_t* n);
  hp_status profile_link(int64_t max, double* link_bytes, int64_t* n);
  hp_status profile_streams(int64_t max, int32_t* ids, int64_t* n);
  int64_t ticks = 0;

 private:
  struct BComplete {
    int v;
    int64_t p;
    int slot;
    bool first, wave_end;
    const float* grad;
    bool snap = false;   // F > 1: snapshot the acc it loads (first backlog completion)
  };
  struct BApply {
    int v;
    int64_t c;
    int slot;
  };
  enum Phase { kNone = 0, kPhComplete = 1, kPhPush = 2, kPhPull = 3 };

  hp_status flush();
  hp_status flush_local();
  hp_status flush_dist();
  // one target of an owner-side pull: the first pulled VW (its w_local) of a
  // (GPU, stage range); the other pulled VWs of that range copy it
  struct Prim {
    int q;
    int64_t a, len;
    int v;
  };
  hp_status dist_accumulate(const std::vector<bool>& pulled);
  hp_status dist_apply(std::vector<Prim>* prims, bool* fuse_pull);
  hp_status dist_pull(const std::vector<Prim>& prims, bool fuse_pull);
  int lockstep_slot() const;                 // acc slot of a lockstep batch, or -1
  hp_status flush_lockstep(int slot);        // its NCCL / NVLS exchange
  hp_status finish_connect(const void* comm_id);
  hp_status xbarrier();
  void prof_begin(cudaStream_t st);
  void prof_end(cudaStream_t st, double bytes, double sync_bytes, int32_t shape,
                double link_bytes = 0);
  hp_status emit(TickDesc& d, int64_t begin, int64_t n, cudaStream_t st = nullptr,
                 int max_blocks = 0, double link_bytes = -1);
  void fork_streams();
  cudaEvent_t pool_event();
  hp_status join_exchange();          // compute stream waits for the exchange stream
  RankLayout layout_of(int q) const;
  int add_segs(TickDesc& d, int64_t a, int64_t len, bool acc_of_vw, int v, int slot);
  hp_status check_cuda(int err, const char* what);
  void rec(char phase, int v, const char* kind, int64_t p, int64_t c);
  std::pair<bool, bool> gate_open(int v) const;
  const float* fold_grad(int v, int64_t p) const;
  // -eta of u(v, p): -lr, or Theorem 1's -sigma/sqrt(t) with t = (p-1)*N + v + 1
  // (hp_config.lr_schedule, reading Z26)
  float neg_lr_of(int v, int64_t p) const;
  // one w_local op of VW v from its pending list: x > 0 FOLD u_x, x < 0 STASH
  // for START(-x) (CONVEX); sets the stash slot / EXTERNAL gradient it reads
  void fill_fold(DFold& f, int v, int64_t x) const;
  bool has_due_folds() const {
    for (const auto& s : vw_)
      if (!s.pending_folds.empty() && !(cfg_.local_semantics == HP_LOCAL_STRICT && s.at_gate)) return true;
    return false;
  }

  hp_config cfg_;
  bool dist_ = false;                 // world > 1: placement with peer exchange
  int G_ = 1, rank_ = 0, span_ = 1;
  std::vector<int64_t> shard_b_;      // PS shard boundaries over G
  std::vector<int64_t> stage_b_;      // VW stage boundaries over span
  std::vector<RankLayout> lay_;
  std::vector<char*> peer_;           // arena base of every rank (own = arena_)
  char* mc_ = nullptr;                // multicast mapping of the arenas (NVLS)
  bool ext_arena_ = false;            // cfg.arena: caller-owned
  std::vector<void*> opened_;         // IPC mappings to close
  Comm* comm_ = nullptr;              // NCCL communicator (nullptr: co-located ranks
                                      // connected without NCCL, hp_connect_symmetric)
  bool connected_ = false;
  // a9 overlap (world > 1): barrier/apply/pull launches run on an exchange
  // stream; a compute-stream launch waits only for the exchange events of the
  // VWs whose buffers it touches.
  cudaStream_t xs_ = nullptr;
  cudaStream_t xs2_ = nullptr;        // second exchange stream (NVLS / peer split)
  int nvls_split_ = 100;              // % of a shard through NVLS (HP_NVLS_SPLIT)
  // Per local VW: accumulation (acc ring) runs on vs_, folds into w_local on
  // fs_ (split_folds_), so the next wave's accumulation does not wait for the
  // pull that rewrites w_local (row a9); exchange ops wait for exactly the
  // producers they read and publish what they freed / wrote.
  std::vector<std::vector<cudaEvent_t>> xacc_;  // [vw][slot]: exchange that last read the slot
  std::vector<cudaEvent_t> xwl_;      // exchange (pull) that last wrote the VW's w_local
  std::vector<cudaEvent_t> lastc_;    // its last acc-writing launch
  std::vector<cudaEvent_t> lastw_;    // its last w_local-writing launch (vs_ or fs_)
  std::vector<cudaStream_t> vs_;      // per local VW: accumulation stream
  std::vector<cudaStream_t> fs_;      // per local VW: fold stream
  bool split_folds_ = false;          // acc and folds in separate launches (HP_SPLIT_FOLDS;
                                      // default rule in finish_connect)
  bool push_pull_ = true;             // owner-side pull (HP_PULL_PUSH=0: reader-side)
  bool forked_ = false;               // side streams ordered after the context stream
  int xblocks_ = 0;                   // grid bound of exchange launches (HP_XBLOCKS)
  int ablocks_ = 0;                   // grid bound of accumulation launches (HP_ABLOCKS)
  bool flag_barrier_ = true;          // K7 device flags (HP_FLAG_BARRIER=0: NCCL barrier)
  uint64_t epoch_ = 0;                // barriers issued (identical on every rank)
  // Point-to-point readiness flags (HP_P2P, default on with the flag
  // barrier): an apply batch waits only for the ranks it involves.
  bool p2p_ = true;
  uint64_t flag_timeout_ns_ = 10000000000ull;   // flag wait deadline (HP_FLAG_TIMEOUT_MS)
  uint64_t xepoch_ = 0;               // apply batches exchanged by flags (replicated)
  uint64_t last_apply_epoch_ = 0;
  std::vector<char> readers_;         // ranks that read w_global shards since the last apply
  unsigned long long* flag_word(int q, int kind, int src) const;   // kind 0 barrier, 1 arrive, 2 done
  hp_status flag_ops(cudaStream_t st, std::vector<unsigned long long*> sig,
                     std::vector<const unsigned long long*> wait, uint64_t val);
  int* flag_err_ = nullptr;           // device: set if a flag wait timed out
  // dynamic tile scheduling of the tick kernel: one (counter, done) pair per
  // launch stream, 128 bytes apart, zero between launches (TickDesc::ctr)
  char* tiles_ = nullptr;
  std::vector<cudaStream_t> tile_streams_;
  bool tile_slot(cudaStream_t st, unsigned long long** ctr, unsigned int** done);
  // HP_STRESS=<seed> (HP_STRESS_US, default 50): before a launch, with
  // probability 1/2, an idle kernel of 0..HP_STRESS_US microseconds on the
  // launch stream (race stress of the stream / event / flag protocol; the
  // arithmetic is unchanged). Per-rank xorshift stream, seeded seed ^ rank.
  uint64_t stress_ = 0;
  uint64_t stress_ns_ = 50000;
  void stress(cudaStream_t st);
  std::vector<cudaEvent_t> evpool_;
  size_t evnext_ = 0;
  double nvl_bytes_ = 0;
  int64_t lockstep_batches_ = 0;
  bool capturing_ = false;            // stream capture of stream_ in progress
  // Multi-tick batching while capturing a small single-rank context
  // (launch_multi_tick): the captured ticks' descriptors are collected and run
  // by one multi-tick kernel per batch; their device copies belong to the graph.
  bool batch_ok_ = false;             // context qualifies (set at init)
  std::vector<TickDescPad> batch_;
  std::vector<void*> graph_bufs_;     // descriptor buffers of the capture in progress
  cudaStream_t up_ = nullptr;         // upload stream (never captured)
  hp_status flush_batch();
 public:
  std::vector<void*> take_graph_bufs() { std::vector<void*> b; b.swap(graph_bufs_); return b; }
 private:
  bool graph_pending_ = false;        // a captured graph awaits its launch
  int64_t apply_batches_ = 0;
  int64_t desc_splits_ = 0;           // launches split because a descriptor table was full
  int N_, Nm_, R_;
  int64_t U_ = 1;                     // minibatches per clock: F * Nm (NEXT-4)
  bool convex_ = false;               // HP_GRAD_CONVEX: stash ring + STASH ops
  int64_t W_, last_p_, n_, begin_;
  cudaStream_t stream_ = nullptr;
  bool own_stream_ = false;
  void* arena_ = nullptr;
  float* wg_ = nullptr;
  float* m_ = nullptr;
  std::vector<VW> vw_;
  std::vector<std::pair<int, int64_t>> commit_;
  std::vector<BApply> pending_applies_;
  int64_t c_global_ = 0, applied_ = 0, tick_ = 0;

  // current batch (one tick)
  Phase phase_ = kNone;
  std::vector<BComplete> bc_;
  std::vector<BApply> ba_;
  std::vector<int> bpull_;              // VWs admitted with a pull in this batch
  std::vector<std::pair<int, int64_t>> ungated_;

  // accounting
  int64_t launches_ = 0;
  double alg_bytes_ = 0;
  bool prof_on_ = false;
  std::vector<cudaEvent_t> ev_;
  size_t ev_used_ = 0;
  double prof_bytes_ = 0;
  std::vector<double> prof_launch_bytes_;
  std::vector<double> prof_launch_sync_;
  std::vector<double> prof_launch_link_;   // NVLink bytes per direction (max of in, out)
  std::vector<int32_t> prof_launch_shape_;
  std::vector<int32_t> prof_launch_stream_;   // 0 context, 1 exchange, 2 second exchange,
                                              // 3+v accumulation of VW v, 3+N+v its fold stream
  int32_t stream_id(cudaStream_t st) const;
  // wave-sync latency: profiled launch that carried VW v's wave-end COMPLETE
  // (its u~ final = the push) -> the launch that wrote its pulled w_local
  std::vector<int64_t> push_launch_;
  struct SyncRec {
    int32_t v;
    int64_t from, to;
    int32_t waited;      // the VW waited at its gate before this pull
  };
  std::vector<SyncRec> sync_recs_;
  void note_sync(const TickDesc& d);
  void note_pulls(const std::vector<int>& vws);
  int64_t prof_launches_ = 0;

  std::string trace_;
  bool trace_on_ = true;
  hp_status sticky_ = HP_OK;
  std::string err_;
};

}  // namespace hp

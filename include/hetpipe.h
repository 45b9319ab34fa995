/*
 * hetpipe.h -- C ABI of the B200-native WSP (Wave Synchronous Parallel) hot path
 * of HetPipe (Park et al., arXiv 2005.14038, USENIX ATC'20).
 *
 * Citations: "P:n" = line n of the paper text (/root/reference/PAPER.md, not
 * shipped); section numbers are the paper's. Readings of silent or ambiguous
 * passages are DESIGN.md "Readings" Z1..Z20.
 *
 * What the library computes (paper sections 4-5):
 *   COMPLETE(v,p)  u_p = fl(-lr * g_p); the open wave's aggregate
 *                  u~ (+)= u_p (summed in completion order, Z1);
 *                  w_local(v) = w_local(v) + u_p, folded "just in
 *                  time" so that minibatch p reads exactly its own updates
 *                  1..p-N_m (STRICT, Z3) or at least those (AT_LEAST).
 *   PUSH(v,c)      at the end of clock c the PS applies w_global = w_global + u~
 *                  (P:928-929), optionally heavy-ball momentum (Z11); c_local(v)
 *                  = c+1, c_global = min over VWs.
 *   GATE/PULL(v)   the next gated minibatch (c+2)*N_m may start iff
 *                  c_local - c_global <= D (Z7); then w_local(v) =
 *                  w_global. LAZY pulls only when the held version is
 *                  older than the bound requires.
 *
 * Layout and ownership:
 *   * All model state lives in device memory owned by the context: w_global and
 *     (momentum) m of this rank's parameter shard, and per VW w_local plus a ring
 *     of acc slots (u~ of waves pushed but not yet applied). fp32, contiguous,
 *     16-byte aligned; the rank owns global params [param_begin, param_begin +
 *     param_count) of every buffer (ED-local placement).
 *   * Param i's synthetic gradient is Philox4x32-10(counter = (i>>2, v, p, 0),
 *     key = (seed lo32, seed hi32)) word i&3, i the GLOBAL index (Z9).
 *   * Device work is stream-ordered and asynchronous on the context's stream;
 *     only hp_sync / hp_read_weights / hp_profile_read block the caller.
 *
 * Errors: every call validates its arguments and the protocol state before it
 * changes anything (no partial effects on error). HP_OK and HP_WOULD_BLOCK are
 * non-errors. A CUDA failure is sticky: every later call returns HP_ERR_CUDA and
 * hp_last_error() holds the text. No C++ exception crosses this ABI. A context
 * is single-threaded (one host controller thread per rank).
 */
#ifndef HETPIPE_H_
#define HETPIPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hp_ctx hp_ctx; /* opaque; owns all device state of one rank */

typedef enum {
  HP_OK = 0,
  HP_WOULD_BLOCK = 1,     /* gate closed: nothing changed */
  HP_ERR_INVALID = -1,    /* bad argument */
  HP_ERR_PROTOCOL = -2,   /* out-of-order / duplicate / incomplete */
  HP_ERR_CUDA = -3,       /* sticky CUDA failure */
  HP_ERR_COMM = -4,       /* inter-GPU transport (NCCL) failure */
  HP_ERR_OOM = -5,        /* device allocation failed */
  HP_ERR_STATE = -6       /* call not valid in this context state */
} hp_status;

/* HP_GRAD_CONVEX: the weight-dependent workload
   g = a (w_p - b) + sigma xi, the gradient of a/2 ||w - b||^2 plus noise at the
   weights w_p = w_local minibatch p read at its START (kept in a ring of N_m
   per-VW stash slots: the "forward pass" of minibatch p); b = Philox stream 2,
   xi = the FLOAT draw; every op one fp32 rounding. */
enum { HP_GRAD_FLOAT = 0, HP_GRAD_DYADIC = 1, HP_GRAD_EXTERNAL = 2, HP_GRAD_CONVEX = 3 };
enum { HP_W0_ZERO = 0, HP_W0_PHILOX = 1 };
enum { HP_PULL_EAGER = 0, HP_PULL_LAZY = 1 };
enum { HP_LOCAL_STRICT = 0, HP_LOCAL_AT_LEAST = 1 };
enum { HP_APPLY_DEFERRED = 0, HP_APPLY_ON_ARRIVAL = 1 };
/* Exchange of a LOCKSTEP batch (world > 1, one full-replica VW per GPU (N = G,
   vw_span 1), SGD, every VW pushing the same wave and pulling in one batch, as
   in D = 0 with equal speeds); every other batch uses PEER:
     PEER  each PS shard owner reads every pushed u~ slice from the GPU that
           holds it inside the apply kernel (NVLink loads, commit order,
           bit-exact), pulls read the w_global shards the same way;
     NCCL  u~ summed per shard by NCCL (grouped ncclReduce, one root per shard =
           reduce-scatter with uneven shards), applied by the owner, w_global
           shards broadcast into every w_local (grouped ncclBroadcast =
           all-gather): the unfused baseline;
     NVLS  one kernel per owner: multimem.ld_reduce of the shard range of every
           GPU's acc slot (the NVSwitch sums), w_global += sum, multimem.st of
           the result into every GPU's w_local (needs the symmetric arena of
           hp_connect_symmetric with a multicast mapping).
   NCCL and NVLS apply the wave's N updates as ONE sum (switch / NCCL order), so
   they match the sequential commit-order apply within rounding (reading Z15,
   normwise <= 1e-5), not bit-exactly; the trace is identical. */
enum { HP_XPORT_PEER = 0, HP_XPORT_NCCL = 1, HP_XPORT_NVLS = 2 };
/* hp_config.lr_schedule */
enum { HP_LR_CONSTANT = 0, HP_LR_THEOREM1 = 1 };

typedef struct {
  int32_t num_vw;          /* N virtual workers, 1..8 */
  int32_t Nm;              /* minibatches per wave, s_local = Nm-1, 1..32 */
  int32_t D;               /* clock-distance threshold, >= 0 */
  int32_t waves;           /* W: minibatches > W*Nm never start (Z16); default 2^30 */
  int64_t nparams;         /* P, global model size */
  int64_t param_begin;     /* first global param owned by this rank (multiple of 32) */
  int64_t param_count;     /* params owned by this rank; -1 = nparams - param_begin */
  float lr;                /* u = fl(-lr*g) (Z2) */
  float momentum;          /* PS heavy-ball mu; 0 = plain SGD apply (Z11) */
  uint64_t seed;           /* Philox key */
  int32_t grad_mode;       /* HP_GRAD_* */
  int32_t w0_mode;         /* HP_W0_* (Z8) */
  int32_t pull_policy;     /* HP_PULL_* (Z6) */
  int32_t local_semantics; /* HP_LOCAL_* (Z3) */
  int32_t apply_mode;      /* HP_APPLY_* (Z4): defer applies to the observing pull */
  int32_t acc_slots;       /* acc ring depth R per VW, 2..8 (default 2) */
  int32_t merge_ticks;     /* 1 (default): ops of consecutive ticks on disjoint VW
                              state may share one launch; 0: one launch per tick */
  int32_t world;           /* G ranks (one process per GPU), 1..8; 1 = single context */
  int32_t rank;            /* this rank, 0..G-1 */
  int32_t vw_span;         /* k GPUs per VW (1..G): VW v's stage j (even split of P
                              over k) lives on GPU (v*k+j) mod G; PS shard q (even
                              split over G) on GPU q. k = G is ED-local (P:104-106,
                              no exchange); k < G exchanges over NVLink. */
  int32_t device;          /* CUDA device ordinal */
  void* stream;            /* cudaStream_t to run on; NULL = library-owned stream */
  int32_t transport;       /* HP_XPORT_* (world > 1): exchange of lockstep batches */
  int32_t reserved;
  int32_t update_freq;     /* F >= 1 (the paper's drafted update
                              frequency factor): one clock = F waves; a VW
                              aggregates and pushes F*Nm minibatches per clock, its gated
                              STARTs are (c+2)*F*Nm, s_global = F(D+2)Nm - 2; `waves`
                              counts clocks. Default 1 */
  int32_t lr_schedule;     /* HP_LR_CONSTANT (default): u = fl(-lr * g). HP_LR_THEOREM1:
                              u(v,p) = fl(-eta_t * g) with eta_t = fl(lr / fl(sqrt(t))),
                              t = (p-1)*num_vw + v + 1 -- Theorem 1's schedule
                              eta_t = sigma/sqrt(t) with lr = sigma, the
                              updates numbered worker-fastest (reading Z26); needs
                              num_vw * waves * F * N_m < 2^24 */
  float conv_a;            /* HP_GRAD_CONVEX curvature a (default 0.5) */
  float conv_sigma;        /* HP_GRAD_CONVEX noise scale sigma (default 1.0) */
  const int64_t* ps_bounds;/* optional PS shard boundaries (world > 1): world+1 values,
                              0 = b[0] < b[1] < ... < b[world] = nparams, inner ones
                              multiples of 32; shard q = [b[q], b[q+1]) on GPU q.
                              NULL = even split (reading Z12; HP_XPORT_NCCL with
                              vw_span 1: ceil split, equal blocks but the last, for
                              the equal-count collectives). Read during
                              hp_init_ex / hp_arena_bytes only (copied). Uneven
                              bounds express e.g. the paper's layer round-robin
                              placement on a permuted parameter order */
  void* arena;             /* optional caller-owned device arena of >= hp_arena_bytes()
                              bytes, 256-byte aligned, BORROWED for the context's
                              lifetime (e.g. a torch symmetric-memory buffer whose peer
                              and multicast mappings go to hp_connect_symmetric);
                              NULL = the library allocates it */
} hp_config;

/* sizeof(hp_config) as compiled into the library (bindings check their layout). */
size_t hp_config_size(void);

/* Fill cfg with defaults (N=1, Nm=1, D=0, lr=0.01, FLOAT grads, PHILOX w0,
   EAGER, STRICT, deferred applies, R=2, merged ticks, device 0, library stream). */
void hp_config_default(hp_config* cfg);

/* Distributed placements (world > 1), set up collectively on every rank:
   rank 0 calls hp_comm_unique_id and broadcasts the 128 bytes; every rank
   calls hp_init_ex, hp_ipc_handle (64 bytes, all-gathered by the caller), then
   hp_connect(handles = world*64 bytes in rank order, comm_id). After that the
   ranks must issue the same protocol calls in the same order (the replicated
   controller does); pushes are applied by each PS shard owner reading the
   pushed u~ slices from the GPU that holds them and storing the new w_global
   into the pullers' w_local (or pulls read w_global shards from their owners)
   -- NVLink loads and stores inside the tick kernels, ordered by a
   stream-ordered barrier: device readiness flags in every arena (release /
   acquire over NVLink; HP_FLAG_BARRIER=0: a 4-byte NCCL
   all-reduce). Each local VW's accumulation, the exchange and (split acc /
   fold launches) the folds run on separate streams: set
   CUDA_DEVICE_MAX_CONNECTIONS >= 16 (e.g. 32) in the environment before the
   process creates its CUDA context, or the runtime's default 8 hardware
   queues serialise them. With a communicator, >= 16 queues, the PEER
   transport, SGD and at most one VW stage per GPU, the accumulation and the
   folds are split into separate launches by default (HP_SPLIT_FOLDS=0/1
   overrides). */
hp_status hp_comm_unique_id(void* out128);
hp_status hp_ipc_handle(hp_ctx* ctx, void* out64);
hp_status hp_connect(hp_ctx* ctx, const void* handles, const void* comm_id);
/* Device bytes of this rank's arena for cfg (the same on every rank of a
   placement whose ranks hold congruent VW sets, e.g. one VW per GPU); < 0 on a
   bad config. */
int64_t hp_arena_bytes(const hp_config* cfg);
/* As hp_connect, for a context whose cfg.arena is a symmetric allocation:
   peer_bases[q] (world entries, q = rank is this arena) is rank q's arena mapped
   into this process, mc_base the multicast mapping of the arenas (NULL if none;
   HP_XPORT_NVLS needs it). No CUDA IPC is used.
   comm_id may be NULL: co-located ranks connected WITHOUT an NCCL communicator
   (e.g. G threads of one process driving G contexts on one GPU, peer_bases =
   the other contexts' arenas). Every barrier is then the K7 device flag
   barrier (HP_FLAG_BARRIER=0 is refused) and the exchange is HP_XPORT_PEER
   (HP_XPORT_NCCL is refused; NVLS without mc_base never runs). The caller
   must let every rank's hp_init_ex return before any rank connects (init
   zeroes the flag arrays); the first flag barrier then orders every rank's
   initialisation before any peer access. Collective: every rank calls it.
   Errors: HP_ERR_STATE (not world > 1, no external arena, already connected,
   or a refused combination above), HP_ERR_COMM (a rank never arrived: the
   flag wait's 10 s deadline). */
hp_status hp_connect_symmetric(hp_ctx* ctx, const void* const* peer_bases, void* mc_base,
                               const void* comm_id);

/* north_star entry point: hp_init(num_vw, Nm, D, nparams, lr) with the other
   fields at their defaults. Allocates ~ (N*(1+R) + 1 (+1 momentum)) * 4 * P
   bytes of device memory and initialises w_global = w_local(v) = w0.
   Errors: HP_ERR_INVALID, HP_ERR_OOM, HP_ERR_CUDA. On error *out = NULL. */
hp_status hp_init(hp_ctx** out, int32_t num_vw, int32_t Nm, int32_t D,
                  int64_t nparams, float lr);
hp_status hp_init_ex(hp_ctx** out, const hp_config* cfg);

/* COMPLETE(vw, p). Requires p == completed(vw)+1 and p
   already started, else HP_ERR_PROTOCOL. grad: HP_GRAD_EXTERNAL only -- device
   fp32[param_count] for this rank's shard (distributed placements: this rank's
   stage of vw, or any non-NULL pointer if vw has no stage here), BORROWED until
   vw's next admission
   (a deferred STRICT fold may re-read it); must be NULL otherwise. If p ends a
   wave the caller must push that wave next (hp_push_wave). The START of
   p+N_m (when not gated) is implicit in this call. */
hp_status hp_accumulate_minibatch(hp_ctx* ctx, int32_t vw, int64_t p, const float* grad);

/* As above with a HOST gradient buffer (pinned for overlap): copied into a
   library-owned device slot on the context stream before the kernel reads it.
   Single-rank contexts: fp32[param_count] (the shard); distributed placements:
   fp32[nparams], the VW's whole gradient, of which this rank copies its stage. */
hp_status hp_accumulate_minibatch_host(hp_ctx* ctx, int32_t vw, int64_t p,
                                       const float* host_grad);

/* PUSH(vw, c): requires c == c_local(vw) and all N_m minibatches of
   wave c completed, else HP_ERR_PROTOCOL (duplicate, out-of-order or
   incomplete push). Appends (vw,c) to the commit log; the PS apply runs in
   commit order, either immediately or deferred to the first pull / read that
   observes w_global (bit-identical either way, Z4). Advances c_local(vw) and
   c_global. */
hp_status hp_push_wave(hp_ctx* ctx, int32_t vw, int64_t c);

/* CLOCK: report c_local(vw) and c_global (either pointer may be NULL). Returns
   HP_WOULD_BLOCK iff vw waits at its gate and the gate is closed. */
hp_status hp_clock(hp_ctx* ctx, int32_t vw, int64_t* c_local, int64_t* c_global);

/* GATE/PULL(vw): only valid while vw waits at its gate (HP_ERR_PROTOCOL
   otherwise). If the gate is closed returns HP_WOULD_BLOCK and changes nothing
   but the trace (first BLOCK). Otherwise pulls per the policy (EAGER always;
   LAZY only if held_g < c_local - D), starts minibatch (c+2)*N_m and replays the
   minibatches that completed while it waited (Z17). Never waits inside. */
hp_status hp_pull(hp_ctx* ctx, int32_t vw);

/* End of a tick: emit the tick's START records (Z5 phase order). Its device ops
   are launched now (merge_ticks = 0) or merged with the next ticks' ops on
   disjoint VW state and launched at the latest by hp_flush / hp_sync /
   hp_read_weights / the return of hp_schedule_advance. */
hp_status hp_tick_end(hp_ctx* ctx);
/* Launch every pending fused op batch and order all launched work (also a
   distributed context's side streams) before later work on the context stream
   (asynchronous; no host sync). */
hp_status hp_flush(hp_ctx* ctx);

/* Stamp subsequent trace records with tick t (wait accounting uses it). */
hp_status hp_set_tick(hp_ctx* ctx, int64_t t);

/* The deterministic tick controller: START(p) for
   p <= N_m at t=0, complete(p) = max(start(p) + lat[v], complete(p-1) + tau[v]);
   phases COMPLETE -> PUSH/APPLY -> GATE/PULL -> START per tick (Z5).
   tau, lat: host int64[num_vw]; lat NULL = N_m * tau. */
hp_status hp_schedule_begin(hp_ctx* ctx, const int64_t* tau, const int64_t* lat);
/* Run ticks until the commit log holds >= target_commits pushes or the run is
   complete; *commits (may be NULL) receives the count reached. Every op of
   those ticks is launched on return. A distributed context's accumulation /
   exchange / fold streams are NOT joined to the context stream here (the next
   call's accumulation may overlap this one's exchange, row a9): call hp_flush
   (or hp_sync) before work on the context stream that must follow them, e.g.
   a timing event. */
hp_status hp_schedule_advance(hp_ctx* ctx, int64_t target_commits, int64_t* commits);
/* CUDA-graph form of hp_schedule_advance, for launch-bound (small) models on
   single-rank contexts (world = 1; a distributed context gets HP_ERR_STATE):
   the controller advances to target_commits NOW on the host (protocol state,
   trace, stats move exactly as hp_schedule_advance), but the device work of
   those ticks -- every fused tick launch -- is captured into one CUDA graph
   (stream capture of the context stream, relaxed mode) instead of running.
   A context of at most HP_TICK_BATCH_MAX_N (default 2^16) params captures its
   ticks as multi-tick launches instead: up to 512 tick descriptors uploaded to
   a device buffer the graph owns, run in order by one kernel each (every
   param's chunk owned by one thread for all ticks, so each tick's loads and
   stores are exactly the per-tick launch's). hp_graph_launch then runs it
   ONCE on the context stream (a graph holds those ticks' descriptors; a
   second launch would redo them, so it is refused: HP_ERR_STATE). Until that
   launch, do not read weights or capture again (HP_ERR_STATE). Launch it
   before hp_finalize of its context. Not allowed with host gradients
   (pageable copies cannot be captured) or while per-launch profiling is on
   (HP_ERR_STATE). *out owned by the caller: hp_graph_destroy (waits for a
   launched graph to finish before freeing its buffers). */
typedef struct hp_graph hp_graph;
hp_status hp_schedule_capture(hp_ctx* ctx, int64_t target_commits, int64_t* commits,
                              hp_graph** out);
hp_status hp_graph_launch(hp_graph* g);
void hp_graph_destroy(hp_graph* g);
/* Calibration for latency-bound configs (C1): device microseconds per launch
   of n back-to-back empty one-CTA kernels on the context stream (launched
   like the tick kernels, with the PDL attribute), issued directly (graph = 0)
   or as one CUDA graph (graph = 1); synchronising. */
hp_status hp_launch_floor(hp_ctx* ctx, int32_t n, int32_t graph, float* us_per_launch);
/* Whole run: begin + advance to num_vw*waves pushes + final apply flush. */
hp_status hp_run_schedule(hp_ctx* ctx, const int64_t* tau, const int64_t* lat);
/* HP_GRAD_EXTERNAL under the controller: COMPLETE(v,p) copies host buffer
   host_bufs[(v*W*F*N_m + p) % n] (each fp32[param_count]; F = update_freq) to
   the device. */
hp_status hp_schedule_set_host_grads(hp_ctx* ctx, const float* const* host_bufs, int32_t n);

/* Wait for all LAUNCHED work (hp_flush, then synchronise the context stream):
   unlike hp_sync, applies deferred to their first observer stay deferred
   (reading Z4), so the batching is the one the run would have had anyway.
   HP_ERR_COMM if a K7 flag wait timed out. */
hp_status hp_drain(hp_ctx* ctx);
/* Flush every pending op and apply, then synchronise the stream. */
hp_status hp_sync(hp_ctx* ctx);

/* Copy count fp32 of a buffer, from local offset `offset`, to host memory.
   which = -1: w_global (pending applies are flushed first); -2: momentum m
   (this rank's PS shard when world > 1); 0..N-1: this rank's stage of
   w_local(which) as its next START will read it (while that VW waits at
   its gate, STRICT folds deferred to admission are not yet in it). Blocking. */
hp_status hp_read_weights(hp_ctx* ctx, int32_t which, int64_t offset, int64_t count,
                          float* host_dst);

/* Version trace, one line per event "t phase vw kind p c c_local c_global a_v
   held_g held_K\n". Writes to path (NULL/"" = keep). */
hp_status hp_trace_dump(hp_ctx* ctx, const char* path);
hp_status hp_trace_enable(hp_ctx* ctx, int32_t enable);

typedef struct {
  int64_t commits;          /* pushes committed */
  int64_t applied;          /* pushes applied on the device */
  int64_t launches;         /* kernel launches issued */
  int64_t ticks;            /* ticks processed by the controller */
  double alg_bytes;         /* algorithmic HBM bytes of all launches */
  int64_t wait_ticks[8];    /* per VW simulated wait */
  int64_t pulls[8];         /* per VW pulls */
  double nvl_bytes;         /* NVLink ingress bytes of this rank's exchange (algorithmic:
                               PEER = its kernels' reads from peer GPUs; NVLS = the
                               switch's reduced u~ + the w_local multicast stores it
                               receives; NCCL = the data the collectives deliver) */
  int64_t lockstep_batches; /* batches exchanged by the NCCL / NVLS transport */
  int64_t apply_batches;    /* PS apply batches (flushes that applied >= 1 push):
                               pushes / apply_batches = the k of SURVEY.md 8(d)'s
                               byte model 16*F*Nm per push + 8(1+[mu]) per batch */
  int64_t desc_splits;      /* extra launches because a tick descriptor table
                               (kMaxC/A/G/F/S, tick_desc.h) was full, plus owner-side
                               pulls refused for more than kMaxP targets */
} hp_stats;
hp_status hp_get_stats(hp_ctx* ctx, hp_stats* out);

/* Per-launch CUDA events on the context stream (enable before the timed region;
   read after it): total kernel ms, algorithmic bytes and launches since enable. */
hp_status hp_profile_enable(hp_ctx* ctx, int32_t enable);
hp_status hp_profile_read(hp_ctx* ctx, double* kernel_ms, double* alg_bytes,
                          int64_t* launches);
/* Per-launch detail of the same window, up to max records: duration (ms),
   algorithmic bytes, and shape = nc | ni<<4 | na<<8 | ng<<16 | nf<<24 | pull<<31
   (completes, inline folds, memory applies, w_local groups, group folds, and
   whether a pull is in the fused launch; nf = 127 marks an NCCL collective of
   HP_XPORT_NCCL: na = 1 the reduce-scatter, ng = 1 the all-gather; nf = 126
   the barrier of a distributed exchange), and
   sync_bytes = the part of
   alg_bytes that is synchronisation (w_global/m traffic, u~ reads of the
   applies, pull writes of w_local; the rest is wave accumulation and folds).
   start_ms = the launch's start relative to the first profiled launch (launches
   of the distributed placements run on several streams and overlap).
   Any output pointer may be NULL. *n = records written. */
hp_status hp_profile_launches(hp_ctx* ctx, int64_t max, float* ms, double* alg_bytes,
                              int32_t* shape, double* sync_bytes, float* start_ms,
                              int64_t* n);

/* Per-launch NVLink bytes of the same window (one entry per hp_profile_launches
   record): the algorithmic bytes per direction (max of in, out) the launch's
   peer / multicast accesses or NCCL collective move through this GPU's links;
   0 for launches that touch only local memory. */
hp_status hp_profile_link(hp_ctx* ctx, int64_t max, double* link_bytes, int64_t* n);
/* Per-launch stream of the same window: 0 = context stream, 1 = exchange
   stream, 2 = second exchange stream (NVLS split), 3+v = accumulation stream
   of VW v, 3+num_vw+v = its fold stream (distributed placements). */
hp_status hp_profile_streams(hp_ctx* ctx, int64_t max, int32_t* stream_ids, int64_t* n);

/* Wave-sync latency of the same window, one record per
   (VW, wave) whose push and pull both fall in it: device time from the start
   of the launch that carried the VW's wave-end COMPLETE (its u~ final: the
   push) to the end of the launch (or NCCL collective) that wrote its pulled
   w_local (a LAZY admission without a pull ends no record; a VW that waited at
   its gate includes the wait and is flagged waited[i] = 1; SURVEY.md 8(d)
   reports the unblocked case). ms[i], vw[i], waited[i] (any may be NULL);
   *n = records written. */
hp_status hp_profile_sync_latency(hp_ctx* ctx, int64_t max, float* ms, int32_t* vw,
                                  int32_t* waited, int64_t* n);

/* ---- Intra-VW pipeline schedule (section 4; no context).
   The upstream generator of the controller's per-VW timing (tau_v, L_v of
   hp_schedule_begin). Times are integer nanoseconds (round-half-even). */
typedef struct {
  int64_t params;        /* parameters of the unit (a layer, or a ResNet block) */
  int64_t fwd_flops;     /* forward FLOPs per sample */
  int64_t act_out;       /* fp32 elements per sample leaving the unit (crosses a cut) */
  int64_t act_resident;  /* fp32 elements per sample kept until its backward pass */
} hp_unit;
typedef struct {
  double flops_per_s;    /* effective training FLOP/s of this GPU */
  double mem_bytes;      /* memory capacity */
  int32_t node;          /* GPUs of one node talk over intra_bps, else inter_bps */
  int32_t reserved;
} hp_gpu;
/* Min-max partition of units[0..L) over the k GPUs of a VW: every
   stage is a contiguous unit range; every GPU order is tried. Stage q (0-based,
   in pipeline order) costs fwd = FLOPs x batch / flops_per_s, bwd = 2 x fwd,
   plus the activation arriving from stage q-1 and the gradient arriving from
   stage q+1 (act_out x 4 x batch over the link between the two GPUs); it must
   fit 3 x 4 x params + min(Nm, 2(k-1-q)+1) x 4 x batch x resident bytes in
   mem_bytes ("the memory requirement will vary depending on the stage",
   P:783). Minimises the largest stage time; ties go to the lexicographically
   smallest (GPU order, cuts). Outputs (each may be NULL): order_out[k] (index
   into gpus of stage q), cuts_out[k+1] (stage q = units [cuts[q], cuts[q+1])),
   stage_costs_out[4k] (fwd, bwd, comm_in_fwd, comm_in_bwd ns per stage),
   *bottleneck_ns. Returns HP_WOULD_BLOCK (not an error) when no split fits the
   memory, HP_ERR_INVALID on bad arguments (k > 8, k > L, ...). */
hp_status hp_partition(const hp_unit* units, int32_t L, const hp_gpu* gpus, int32_t k,
                       int32_t Nm, int32_t batch, double intra_bps, double inter_bps,
                       int32_t* order_out, int32_t* cuts_out, int64_t* stage_costs_out,
                       int64_t* bottleneck_ns);
/* Max_m: the largest Nm in [1, 2k-1] with a feasible partition, 0
   if even Nm = 1 does not fit. */
int32_t hp_max_m(const hp_unit* units, int32_t L, const hp_gpu* gpus, int32_t k, int32_t batch,
                 double intra_bps, double inter_bps);
/* Event-driven pipeline of one VW over P minibatches: per GPU
   forward tasks in minibatch order (condition 1), backward tasks in minibatch
   order (2), FIFO among ready tasks (3; ties: backward first, lower minibatch
   first); the last stage runs forward+backward as one task; minibatch p
   starts at 0 if p <= Nm, else when p-Nm completes (local staleness Nm-1,
   P:817); p completes when its backward pass leaves stage 0 (u_p exists).
   stage_costs[4k] as hp_partition's output. start_out/complete_out: int64[P]
   (either may be NULL). */
hp_status hp_pipeline_simulate(const int64_t* stage_costs, int32_t k, int32_t Nm, int64_t P,
                               int64_t* start_out, int64_t* complete_out);
/* The tick model's two numbers from that simulation (reading Z13): tau = the
   mean completion interval over the middle half of a P-minibatch run (P <= 0:
   24 Nm; floor), latency = minibatch 1's start-to-complete time. */
hp_status hp_pipeline_tau_latency(const int64_t* stage_costs, int32_t k, int32_t Nm, int64_t P,
                                  int64_t* tau_ns, int64_t* latency_ns);

/* Closed forms of section 5 (no context needed). */
int64_t hp_s_global(int32_t Nm, int32_t D);                  /* (D+1)*Nm + Nm - 2 */
int64_t hp_s_global_f(int32_t Nm, int32_t D, int32_t F);     /* F(D+2)Nm - 2 */
int64_t hp_version_floor(int64_t p, int32_t Nm, int32_t D);  /* max(0, p - s_global - 1) */

const char* hp_last_error(const hp_ctx* ctx);   /* NULL ctx: last init error */
const char* hp_version(void);
void hp_finalize(hp_ctx* ctx);                  /* frees everything; NULL ok */

#ifdef __cplusplus
}
#endif
#endif /* HETPIPE_H_ */

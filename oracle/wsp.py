"""WSP (Wave Synchronous Parallel) oracle: the protocol of PAPER.md sections 4-5,
run step by step on a deterministic tick schedule.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation follows the paper: N virtual workers (VWs), N_m minibatches per wave,
s_local = N_m - 1, clock-distance threshold D, local clock
c_local per VW and global clock c_global = min c_local. Every
floating-point step is one float32 numpy operation (round-to-nearest-even, no
FMA), in the order the paper states it. Where the paper is silent the reading
taken is the one listed in DESIGN.md "Readings" (Z-numbers from SURVEY.md 8(c)).

Method summary with citations:
  * COMPLETE(v,p): u_p = -lr * g(v,p) (Z2);  "w_local = w_local + u_p"
    and the wave aggregate u~ = sum of u over minibatches c*N_m+1 .. (c+1)*N_m
    (P:922), summed in completion order (Z1: sum, not average).
  * PUSH(v,c) at the end of clock c: the PS applies "w_global = w_global + u~"
     on arrival (Z4); c_local = c+1 and c_global = min c_local, so
    c_global moves to c+1 only after every VW pushed wave c.
  * GATE at the end of clock c for the next gated minibatch (c+2)*N_m (the one
    the paper's D=0 example waits on, minibatch 8 for N_m=4): the VW
    may proceed iff c_local - c_global <= D (Z7), then pulls w_global
    (EAGER; LAZY pulls only when its held version is too old);
    while it waits, the s_local minibatches already in flight keep completing
    (Z17).
  * START(v,p) reads w_local; STRICT semantics (Z3) make the own updates in it
    exactly 1..p-N_m ("at least", north_star "never newer").
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from workloads import (GRAD_CONVEX, GRAD_DYADIC, GRAD_FLOAT, LOCAL_AT_LEAST, LOCAL_STRICT,
                       PULL_EAGER, PULL_LAZY, W0_PHILOX, W0_ZERO, WSPConfig)

from .philox import philox4x32_10

F32 = np.float32


# --------------------------------------------------------------------------- #
# Closed forms of section 5                                                    #
# --------------------------------------------------------------------------- #
def wave_range(c: int, Nm: int) -> Tuple[int, int]:
    """Minibatches of wave c: c*(s_local+1)+1 .. (c+1)*(s_local+1)."""
    return c * Nm + 1, (c + 1) * Nm


def s_global(Nm: int, D: int, F: int = 1) -> int:
    """s_global = (D+1)*(s_local+1) + s_local - 1, s_local = Nm-1;
    with the update frequency factor F (one clock = F waves):
    F*(D+1)*(s_local+1) + (F-1)*(s_local+1) + s_local - 1 = F*(D+2)*(s_local+1) - 2."""
    s_local = Nm - 1
    return F * (D + 1) * (s_local + 1) + (F - 1) * (s_local + 1) + s_local - 1


def version_floor(p: int, Nm: int, D: int, F: int = 1) -> int:
    """Minibatch p must reflect the global updates of minibatches 1..p-(s_global+1)
    (P:998); 0 inside the initial region p <= (D+1)(s_local+1)+s_local."""
    return max(0, p - (s_global(Nm, D, F) + 1))


def wave_of(p: int, Nm: int) -> int:
    return (p - 1) // Nm


def clock_range(c: int, U: int) -> Tuple[int, int]:
    """Minibatches aggregated by clock c: c*F*(s_local+1)+1 .. (c+1)*F*(s_local+1)
    (P:1086-1087), U = F*Nm (= wave_range for F = 1)."""
    return c * U + 1, (c + 1) * U


# --------------------------------------------------------------------------- #
# Synthetic gradients and initial weights (stand-in for the backward pass)     #
# --------------------------------------------------------------------------- #
def _draws(idx: np.ndarray, vw: int, p: int, stream: int, seed: int) -> np.ndarray:
    """uint32 draw of each param in idx: Philox4x32-10, counter (i>>2, vw, p,
    stream), key (seed lo32, seed hi32), word i&3."""
    blk = idx >> 2
    ublk, inv = np.unique(blk, return_inverse=True)
    words = philox4x32_10(ublk.astype(np.uint64), np.uint64(vw), np.uint64(p),
                          np.uint64(stream), seed & 0xFFFFFFFF,
                          (seed >> 32) & 0xFFFFFFFF)
    table = np.stack(words, axis=1)                     # [n_unique_blocks, 4]
    return table[inv, idx & 3]


def gradient(idx: np.ndarray, vw: int, p: int, cfg: WSPConfig,
             w: Optional[np.ndarray] = None) -> np.ndarray:
    """g(v,p,i) as float32. FLOAT: (x>>8)*2^-24 - 0.5 (exact, in [-0.5,0.5));
    DYADIC: (x>>28) - 8 (integers -8..7). CONVEX (NEXT-2, the weight-dependent
    workload of SURVEY.md 8(f)): the gradient of f(w) = a/2 ||w - b||^2 at the
    weights w = w_p minibatch p read at its START, plus noise:
    g = fl(fl(a * fl(w - b)) + fl(sigma * xi)), xi = the FLOAT draw."""
    x = _draws(idx, vw, p, 0, cfg.seed)
    if cfg.grad_mode == GRAD_FLOAT:
        return ((x >> 8).astype(np.float64) * 2.0 ** -24 - 0.5).astype(F32)
    if cfg.grad_mode == GRAD_DYADIC:
        return ((x >> 28).astype(np.int64) - 8).astype(F32)
    if cfg.grad_mode == GRAD_CONVEX:
        assert w is not None, "CONVEX gradients need w_p"
        xi = ((x >> 8).astype(np.float64) * 2.0 ** -24 - 0.5).astype(F32)
        d = w - convex_target(idx, cfg)
        return (F32(cfg.conv_a) * d) + (F32(cfg.conv_sigma) * xi)
    raise ValueError("oracle supports FLOAT, DYADIC and CONVEX gradients only")


def convex_target(idx: np.ndarray, cfg: WSPConfig) -> np.ndarray:
    """b of the CONVEX workload: Philox stream 2, counter (i>>2, 0, 0, 2),
    2*((x>>8)*2^-24) - 1 in [-1, 1) (exact in float32)."""
    x = _draws(idx, 0, 0, 2, cfg.seed)
    return (2.0 * ((x >> 8).astype(np.float64) * 2.0 ** -24) - 1.0).astype(F32)


def initial_weights(idx: np.ndarray, cfg: WSPConfig) -> np.ndarray:
    """w0 ("w_0 ... is given"): zero, or Philox stream 1 with counter
    (i>>2, 0, 0, 1): FLOAT 2*((x>>8)*2^-24) - 1, DYADIC (x>>25)*2^-6 - 1 (Z8)."""
    if cfg.w0_mode == W0_ZERO:
        return np.zeros(idx.size, dtype=F32)
    x = _draws(idx, 0, 0, 1, cfg.seed)
    if cfg.grad_mode == GRAD_DYADIC:
        return ((x >> 25).astype(np.float64) * 2.0 ** -6 - 1.0).astype(F32)
    return (2.0 * ((x >> 8).astype(np.float64) * 2.0 ** -24) - 1.0).astype(F32)


def step_size(vw: int, p: int, cfg: WSPConfig) -> np.float32:
    """eta of minibatch p of VW vw: the constant lr (Z2), or Theorem 1's
    schedule eta_t = sigma / sqrt(t) (App. A)
    with sigma = cfg.lr and the updates numbered worker-fastest,
    t = (p - 1) * N + vw + 1 (the loop "over the workers (t mod N)" of P:1511-1515;
    reading Z26). float32: fl(sigma / fl(sqrt(t))), t exact."""
    if getattr(cfg, "lr_schedule", 0) == 0:
        return F32(cfg.lr)
    t = F32((p - 1) * cfg.num_vw + vw + 1)
    return F32(cfg.lr) / np.sqrt(t)


def update(idx: np.ndarray, vw: int, p: int, cfg: WSPConfig,
           w: Optional[np.ndarray] = None) -> np.ndarray:
    """u_p = fl(-eta * g_p): one float32 rounding (Z2, Z10); eta = step_size."""
    return (-step_size(vw, p, cfg)) * gradient(idx, vw, p, cfg, w)


# --------------------------------------------------------------------------- #
# The protocol state machine                                                   #
# --------------------------------------------------------------------------- #
class WSPOracle:
    """State of N VWs and the parameter server over a param index subset `idx`
    (every step is element-wise in the param index, so any subset of the full
    run is computed exactly by restricting to it)."""

    def __init__(self, cfg: WSPConfig, idx: Optional[np.ndarray] = None,
                 record_snapshots: bool = False):
        self.cfg = cfg
        self.idx = (np.arange(cfg.nparams, dtype=np.int64) if idx is None
                    else np.asarray(idx, dtype=np.int64))
        N = cfg.num_vw
        w0 = initial_weights(self.idx, cfg)
        self.wg = w0.copy()                                  # w_global
        self.m = np.zeros_like(w0)                           # PS momentum (Z11)
        self.wl = [w0.copy() for _ in range(N)]              # w_local
        self.acc = [np.zeros_like(w0) for _ in range(N)]     # u~ of the open wave
        self.acc_count = [0] * N                             # completions in it
        self.c_local = [0] * N                               # P:919 initially 0
        self.c_global = 0
        self.commit: List[Tuple[int, int]] = []              # PS apply order
        self.started = [0] * N
        self.completed = [0] * N
        self.a = [0] * N                                     # own-update cursor a_v
        self.held_g = [0] * N
        self.held_K = [0] * N
        self.at_gate = [False] * N                           # pushed, not yet admitted
        self.blocked = [False] * N
        self.t_block = [0] * N
        self.backlog: List[List[int]] = [[] for _ in range(N)]
        self.wait = [0] * N
        self.pulls = [0] * N
        self.trace: List[str] = []
        self.record_snapshots = record_snapshots
        self.snapshots: List[Tuple[int, int, int, np.ndarray]] = []
        self.start_versions: List[Tuple[int, int, int, int]] = []  # (v, p, a_v, held_K)
        # CONVEX: w_p, the w_local minibatch p read at its START, until u_p's
        # last use (its COMPLETE and its fold)
        self.w_at_start: List[Dict[int, np.ndarray]] = [dict() for _ in range(N)]
        # F > 1, STRICT: the aggregate of the VW's own unpushed updates when it
        # reached its gate, kept if later completions (the backlog) join acc
        self.acc_at_gate: List[Optional[np.ndarray]] = [None] * N

    # -- helpers ---------------------------------------------------------------
    @property
    def U(self) -> int:
        """Minibatches per clock: F waves of Nm (F = 1: one wave)."""
        return self.cfg.F * self.cfg.Nm

    @property
    def last_p(self) -> int:
        return self.cfg.waves * self.U

    def _rec(self, t: int, phase: str, v: int, kind: str, p: int, c: int) -> None:
        self.trace.append(f"{t} {phase} {v} {kind} {p} {c} {self.c_local[v]} "
                          f"{self.c_global} {self.a[v]} {self.held_g[v]} "
                          f"{self.held_K[v]}")

    def _u(self, v: int, p: int) -> np.ndarray:
        return update(self.idx, v, p, self.cfg, self.w_at_start[v].get(p))

    def _folded(self, v: int, p: int) -> None:
        """u_p's fold happened (its COMPLETE came first): w_p is dead."""
        self.w_at_start[v].pop(p, None)

    # -- events ----------------------------------------------------------------
    def start(self, t: int, v: int, p: int, phase: str = "S") -> None:
        """START(v,p): minibatch p reads the latest w_local."""
        cfg = self.cfg
        assert p == self.started[v] + 1 and p <= self.last_p, (v, p)
        if cfg.local_semantics == LOCAL_STRICT:
            assert self.a[v] == max(0, p - cfg.Nm), (v, p, self.a[v])   # Z3
        self.started[v] = p
        self._rec(t, phase, v, "START", p, wave_of(p, self.U))
        self.start_versions.append((v, p, self.a[v], self.held_K[v]))
        if cfg.grad_mode == GRAD_CONVEX:
            self.w_at_start[v][p] = self.wl[v].copy()     # the forward pass reads w_p
        if self.record_snapshots:
            self.snapshots.append((t, v, p, self.wl[v].copy()))

    def complete(self, t: int, v: int, p: int) -> Tuple[bool, bool]:
        """COMPLETE(v,p). Returns (clock_end, ungated_start_of_p+Nm)."""
        cfg = self.cfg
        Nm, U = cfg.Nm, self.U
        assert p == self.completed[v] + 1 and p <= self.started[v], (v, p)
        self.completed[v] = p
        u = self._u(v, p)
        if self.at_gate[v] and not self.backlog[v] and self.acc_count[v]:
            self.acc_at_gate[v] = self.acc[v].copy()     # before the backlog joins
        if (p - 1) % U == 0:                     # first minibatch of its clock
            self.acc[v] = u.copy()
            self.acc_count[v] = 1
        else:
            self.acc[v] = self.acc[v] + u        # aggregated updates
            self.acc_count[v] += 1
        wave_end = p % U == 0
        # START(p+Nm) is the gated one iff p+Nm = (c+2)*U (with F:
        # "continues to execute up to (F-1)(s_local+1) + s_local minibatches")
        gated_next = (p + Nm) % U == 0 and 2 * U <= p + Nm <= self.last_p
        start_next = False
        if not self.at_gate[v]:
            self.wl[v] = self.wl[v] + u          # w_local = w_local + u_p
            self.a[v] = p
            self._folded(v, p)
            if gated_next:
                self.at_gate[v] = True           # evaluated in this tick's GATE phase
                self.acc_at_gate[v] = None
            start_next = (not gated_next) and p + Nm <= self.last_p
        else:                                    # waiting at the gate (Z17)
            self.backlog[v].append(p)
            if cfg.local_semantics == LOCAL_AT_LEAST:
                self.wl[v] = self.wl[v] + u
                self.a[v] = p
                self._folded(v, p)
        self._rec(t, "C", v, "COMPLETE", p, wave_of(p, U))
        return wave_end, start_next

    def push(self, t: int, v: int, c: int) -> None:
        """PUSH(v,c) and the PS apply on arrival (Z4, Z11)."""
        cfg = self.cfg
        assert c == self.c_local[v], "out-of-order or duplicate push"
        assert self.completed[v] == (c + 1) * self.U, "incomplete wave"
        ut = self.acc[v]
        if cfg.momentum == 0.0:
            self.wg = self.wg + ut                         # w_global = w_global + u~
        else:
            self.m = (F32(cfg.momentum) * self.m) + ut     # m = mu*m + u~
            self.wg = self.wg + self.m
        self.commit.append((v, c))
        self.c_local[v] = c + 1
        self.c_global = min(self.c_local)
        self.acc_count[v] = 0
        self._rec(t, "P", v, "PUSH", (c + 1) * self.U, c)

    def gate_open(self, v: int) -> Tuple[bool, bool]:
        """(admissible, needs_pull) for the VW waiting at its gate."""
        cfg = self.cfg
        within = self.c_local[v] - self.c_global <= cfg.D
        if cfg.pull_policy == PULL_EAGER:
            return within, True
        if self.held_g[v] >= self.c_local[v] - cfg.D:      # held version is enough
            return True, False
        return within, True

    def pull(self, t: int, v: int) -> None:
        """w_local <- w_global (STRICT) or w_global + partial u~ (AT_LEAST)."""
        cfg = self.cfg
        if cfg.local_semantics == LOCAL_STRICT:
            # own updates up to p - Nm of the gated p = (c_local+1)*U: the pushed
            # ones are in w_global; with F > 1 those of the open clock are added
            # as their aggregate (reading Z25)
            gate_a = (self.c_local[v] + 1) * self.U - cfg.Nm
            if gate_a > self.c_local[v] * self.U:
                part = self.acc_at_gate[v] if self.backlog[v] else self.acc[v]
                self.wl[v] = self.wg + part
            else:
                self.wl[v] = self.wg.copy()
            self.a[v] = gate_a
        else:
            self.wl[v] = (self.wg + self.acc[v]) if self.acc_count[v] else self.wg.copy()
            self.a[v] = self.completed[v]
        self.held_g[v] = self.c_global
        self.held_K[v] = len(self.commit)
        self.pulls[v] += 1

    def try_admit(self, t: int, v: int) -> List[int]:
        """GATE/PULL phase for v. Returns the minibatches started (in order)."""
        cfg = self.cfg
        ok, needs_pull = self.gate_open(v)
        c = self.c_local[v] - 1
        gated_p = (self.c_local[v] + 1) * self.U             # (c+2)*U
        if not ok:
            if not self.blocked[v]:
                self.blocked[v] = True
                self.t_block[v] = t
                self._rec(t, "G", v, "BLOCK", gated_p, c)
            return []
        if self.blocked[v]:
            self.wait[v] += t - self.t_block[v]
            self.blocked[v] = False
        self.at_gate[v] = False
        if needs_pull:
            self.pull(t, v)
            self._rec(t, "G", v, "PULL", gated_p, c)
        else:
            self._rec(t, "G", v, "ADMIT", gated_p, c)
        started = []
        self.start(t, v, gated_p, phase="G")
        started.append(gated_p)
        for q in self.backlog[v]:                            # Z17 replay in order
            if cfg.local_semantics == LOCAL_STRICT:
                self.wl[v] = self.wl[v] + self._u(v, q)      # deferred fold (Z3)
                self.a[v] = q
                self._folded(v, q)
                self._rec(t, "G", v, "FOLD", q, wave_of(q, self.U))
            if q + cfg.Nm <= self.last_p:
                self.start(t, v, q + cfg.Nm, phase="G")
                started.append(q + cfg.Nm)
        self.backlog[v] = []
        return started

    def done(self) -> bool:
        return all(c == self.cfg.waves for c in self.c_local)


# --------------------------------------------------------------------------- #
# Tick driver                                                                  #
# --------------------------------------------------------------------------- #
@dataclasses.dataclass
class OracleRun:
    trace: List[str]
    wg: np.ndarray
    m: np.ndarray
    wl: List[np.ndarray]
    commit: List[Tuple[int, int]]
    wait: List[int]
    pulls: List[int]
    snapshots: List[Tuple[int, int, int, np.ndarray]]
    start_versions: List[Tuple[int, int, int, int]]
    ticks: List[int]
    max_clock_gap: int


def run_schedule(cfg: WSPConfig, idx: Optional[np.ndarray] = None,
                 record_snapshots: bool = False,
                 on_tick=None) -> OracleRun:
    """Run the WSP protocol for cfg.waves waves per VW on the tick model (Z13):
    START(p) for p <= N_m at t=0; complete(p) = max(start(p) + L_v,
    complete(p-1) + tau_v). Events of one tick are processed in the phases
    COMPLETE -> PUSH/APPLY -> GATE/PULL -> START, ascending VW within a phase
    (Z5). `on_tick(t, oracle)` is called after every tick (parity tests)."""
    sm = WSPOracle(cfg, idx, record_snapshots)
    N, Nm = cfg.num_vw, cfg.Nm
    tau, lat = cfg.tau, cfg.latency()
    ctime: List[Dict[int, int]] = [dict() for _ in range(N)]
    pending: Dict[int, List[Tuple[int, int]]] = {}

    def schedule(t: int, v: int, p: int) -> None:
        ct = t + lat[v]
        if p - 1 in ctime[v]:
            ct = max(ct, ctime[v][p - 1] + tau[v])
        ctime[v][p] = ct
        pending.setdefault(ct, []).append((v, p))

    for v in range(N):
        for p in range(1, min(Nm, sm.last_p) + 1):
            sm.start(0, v, p)
            schedule(0, v, p)
    ticks = []
    max_gap = 0
    while not sm.done():
        assert pending, "deadlock: no pending completion"
        t = min(pending)
        comps = sorted(pending.pop(t))
        ticks.append(t)
        pushes, ungated = [], []
        for v, p in comps:                                   # COMPLETE phase
            wave_end, start_next = sm.complete(t, v, p)
            if wave_end:
                pushes.append((v, wave_of(p, sm.U)))
            if start_next:
                ungated.append((v, p + Nm))
        for v, c in pushes:                                  # PUSH/APPLY phase
            sm.push(t, v, c)
        max_gap = max(max_gap, max(sm.c_local) - min(sm.c_local))
        for v in range(N):                                   # GATE/PULL phase
            if sm.at_gate[v]:
                for p in sm.try_admit(t, v):
                    schedule(t, v, p)
        for v, p in ungated:                                 # START phase
            sm.start(t, v, p)
            schedule(t, v, p)
        if on_tick is not None:
            on_tick(t, sm)
    return OracleRun(sm.trace, sm.wg, sm.m, sm.wl, sm.commit, sm.wait, sm.pulls,
                     sm.snapshots, sm.start_versions, ticks, max_gap)

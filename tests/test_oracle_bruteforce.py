"""P13: brute force over every admissible interleaving of 2 VW x 3 waves x 8
params (north_star), DYADIC gradients so fp32 is exact.

Atomic per-VW steps (untimed model):
  COMPLETE(v): complete the next started minibatch; at a wave end this includes
               the PUSH; if v is not waiting at its gate, START(p+N_m) too.
  ADMIT(v):    enabled iff v waits at its gate and the gate holds;
               gate + pull + gated START + backlog replay.
Every reachable state is checked once (memoised DFS over the state, which fixes
the arrays); the number of complete paths is counted by dynamic programming.
For each transition: every START snapshot equals w0 + the other VWs' pushed
waves in the held commit prefix + own updates 1..a_v, recomputed from scratch,
a_v = p - N_m exactly (STRICT), and the clock distance stays <= D+1; every
terminal state has w_global = w0 + all updates (P9)."""
import copy

import numpy as np
import pytest

from oracle.wsp import WSPOracle, clock_range, gradient, initial_weights, wave_range
from workloads import (GRAD_DYADIC, LOCAL_AT_LEAST, LOCAL_STRICT, PULL_EAGER,
                       PULL_LAZY, W0_PHILOX, WSPConfig)


def _key(sm):
    return (tuple(sm.started), tuple(sm.completed), tuple(sm.c_local),
            tuple(sm.a), tuple(sm.held_g), tuple(sm.held_K), tuple(sm.at_gate),
            tuple(tuple(b) for b in sm.backlog), tuple(sm.commit))


def explore(cfg, seen=None):
    idx = np.arange(8)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    CU = cfg.F * cfg.Nm                    # minibatches per clock (F waves)
    U = {(v, p): -float(np.float32(cfg.lr)) * gradient(idx, v, p, cfg).astype(np.float64)
         for v in range(cfg.num_vw) for p in range(1, cfg.waves * CU + 1)}

    mu = cfg.momentum

    def version(v, a_v, prefix):
        if mu:
            return heavy_ball(v, a_v, prefix)
        tot = w0.copy()
        for q in range(1, a_v + 1):
            tot += U[(v, q)]
        for (vv, c) in prefix:
            if vv != v:
                lo, hi = clock_range(c, CU)
                for q in range(lo, hi + 1):
                    tot += U[(vv, q)]
        return tot

    def heavy_ball(v, a_v, prefix):
        """Z11 in closed form over the commit order: w0 + sum_j u~_(j)
        (1 - mu^(K-j+1)) / (1 - mu), + own updates not in a pushed clock of the
        prefix, up to a_v (exact for mu = 1/2 and DYADIC terms)."""
        K = len(prefix)
        tot = w0.copy()
        own = set()
        for j, (vv, c) in enumerate(prefix, start=1):
            lo, hi = clock_range(c, CU)
            for q in range(lo, hi + 1):
                tot += U[(vv, q)] * (1 - mu ** (K - j + 1)) / (1 - mu)
            if vv == v:
                own.update(range(lo, hi + 1))
        for q in range(1, a_v + 1):
            if q not in own:
                tot += U[(v, q)]
        return tot

    root = WSPOracle(cfg, idx, record_snapshots=True)
    for v in range(cfg.num_vw):
        for p in range(1, min(cfg.Nm, root.last_p) + 1):
            root.start(0, v, p)
    memo = {}
    stats = {"states": 0, "starts": 0, "max_gap": 0}

    def enabled(sm):
        steps = []
        for v in range(cfg.num_vw):
            if sm.completed[v] < sm.started[v]:
                steps.append(("C", v))
            if sm.at_gate[v] and sm.gate_open(v)[0]:
                steps.append(("A", v))
        return steps

    def apply(sm, step):
        kind, v = step
        if kind == "C":
            p = sm.completed[v] + 1
            wave_end, start_next = sm.complete(0, v, p)
            if wave_end:
                sm.push(0, v, (p - 1) // CU)
            if start_next:
                sm.start(0, v, p + cfg.Nm)
        else:
            sm.try_admit(0, v)

    def check(sm, n_snap_before):
        for (t, v, p, snap), (v2, p2, a_v, held_K) in zip(
                sm.snapshots[n_snap_before:], sm.start_versions[n_snap_before:]):
            assert (v, p) == (v2, p2)
            if cfg.local_semantics == LOCAL_STRICT:
                assert a_v == max(0, p - cfg.Nm)
            assert np.array_equal(snap.astype(np.float64),
                                  version(v, a_v, sm.commit[:held_K]))
            stats["starts"] += 1
            if seen is not None:      # newest other-VW minibatch this START holds
                top = min(max([clock_range(c, CU)[1] for vv, c in sm.commit[:held_K]
                               if vv == o], default=0)
                          for o in range(cfg.num_vw) if o != v)
                seen[(v, p)] = min(seen.get((v, p), top), top)
        gap = max(sm.c_local) - min(sm.c_local)
        assert gap <= cfg.D + 1
        stats["max_gap"] = max(stats["max_gap"], gap)

    def count(sm):
        k = _key(sm)
        if k in memo:
            return memo[k]
        stats["states"] += 1
        steps = enabled(sm)
        if not steps:
            assert sm.done(), "stuck state"
            allp = [(v, q) for v in range(cfg.num_vw) for q in range(1, sm.last_p + 1)]
            tot = w0.copy()
            for vq in allp:
                tot += U[vq]
            if mu:
                tot = heavy_ball(-1, 0, sm.commit)
            assert np.array_equal(sm.wg.astype(np.float64), tot)
            memo[k] = 1
            return 1
        total = 0
        for st in steps:
            nxt = copy.deepcopy(sm)
            n0 = len(nxt.snapshots)
            apply(nxt, st)
            check(nxt, n0)
            # drop history that the key does not cover, to keep copies small
            nxt.snapshots, nxt.start_versions, nxt.trace = [], [], []
            total += count(nxt)
        memo[k] = total
        return total

    n = count(root)
    return n, stats


def _cfg(Nm, D, policy=PULL_EAGER, sem=LOCAL_STRICT, momentum=0.0):
    return WSPConfig("bf", 2, Nm, D, 8, 3, (1, 1), lr=2.0 ** -6,
                     grad_mode=GRAD_DYADIC, w0_mode=W0_PHILOX,
                     pull_policy=policy, local_semantics=sem, momentum=momentum)


@pytest.mark.parametrize("D,expected", [(0, 72), (1, 240), (2, 252), (3, 252)])
def test_bruteforce_nm1(D, expected):
    """N_m=1: D>=2 leaves the two 5-step sequences unconstrained, C(10,5)=252
    (closed form); D=0/1 counts cross-check SURVEY.md 0.4 [scratch] 6."""
    n, _ = explore(_cfg(1, D))
    assert n == expected


@pytest.mark.parametrize("D,expected", [(0, 70400), (1, 200704), (2, 205920)])
def test_bruteforce_nm2(D, expected):
    """N_m=2, 2 VW x 3 waves x 8 params; counts cross-check SURVEY.md [scratch] 6."""
    n, stats = explore(_cfg(2, D))
    assert n == expected
    assert stats["starts"] > 0


@pytest.mark.parametrize("policy,sem", [(PULL_LAZY, LOCAL_STRICT),
                                        (PULL_EAGER, LOCAL_AT_LEAST),
                                        (PULL_LAZY, LOCAL_AT_LEAST)])
@pytest.mark.parametrize("D", [0, 1])
def test_bruteforce_policies(policy, sem, D):
    """The same exact version-set checks under LAZY pulls and the
    paper-literal AT_LEAST local semantics. LAZY admits without a
    pull when the held version suffices, so the path set is the same."""
    n, _ = explore(_cfg(2, D, policy, sem))
    assert n == {0: 70400, 1: 200704}[D]


@pytest.mark.parametrize("Nm,D,expected", [(1, 0, 72), (1, 1, 240), (2, 0, 70400),
                                           (2, 1, 200704)])
@pytest.mark.parametrize("policy,sem", [(PULL_EAGER, LOCAL_STRICT),
                                        (PULL_LAZY, LOCAL_AT_LEAST)])
def test_bruteforce_momentum(Nm, D, expected, policy, sem):
    """P15 on every interleaving: with heavy-ball momentum mu = 1/2 (Z11; exact
    in fp32 on DYADIC terms) every START snapshot and the final w_global equal
    the heavy-ball closed form over that interleaving's commit order (+ own
    unpushed updates); the path set is the one of plain SGD."""
    n, stats = explore(_cfg(Nm, D, policy, sem, momentum=0.5))
    assert n == expected and stats["starts"] > 0


@pytest.mark.parametrize("D,expected", [(0, 22415400), (1, 56362878), (2, 57139992)])
def test_bruteforce_nm3(D, expected):
    """N_m=3 (memoised state space); counts cross-check SURVEY.md [scratch] 6
    (22.4M / 56.4M / 57.1M)."""
    n, _ = explore(_cfg(3, D))
    assert n == expected


@pytest.mark.parametrize("Nm,D,sem", [(1, 0, LOCAL_STRICT), (1, 1, LOCAL_STRICT),
                                      (2, 0, LOCAL_STRICT), (2, 1, LOCAL_AT_LEAST)])
def test_bruteforce_update_frequency(Nm, D, sem):
    """NEXT-4 (F = 2 waves per clock): every admissible
    interleaving of 2 VW x 2 clocks keeps START snapshots = version-set sums,
    a_v = p - Nm (STRICT) and the clock bound; gates only at (c+2) F Nm."""
    cfg = WSPConfig("bf", 2, Nm, D, 8, 2, (1, 1), lr=2.0 ** -6, grad_mode=GRAD_DYADIC,
                    w0_mode=W0_PHILOX, local_semantics=sem, F=2)
    n, stats = explore(cfg)
    assert n > 0 and stats["starts"] > 0


def test_bruteforce_update_frequency_counts():
    """F = 2, Nm = 1, 2 clocks: each VW runs C1, C2 (push of clock 0), C3 (it
    reaches the gate of minibatch (0+2)*F*Nm = 4), ADMIT, C4 (push of clock 1).
    With D = 0 its ADMIT needs the other VW's clock-0 push (c_local - c_global
    <= 0); with D = 1 nothing binds. Counted here directly over merges of
    the two 5-step sequences (independent of the oracle) and compared with the
    oracle's exhaustive exploration."""
    import itertools
    for D in (0, 1):
        n = 0
        for xs in itertools.combinations(range(10), 5):   # positions of VW 0's steps
            ys = [i for i in range(10) if i not in xs]
            ok = D >= 1 or (xs[3] > ys[1] and ys[3] > xs[1])
            n += ok
        cfg = WSPConfig("bf", 2, 1, D, 8, 2, (1, 1), lr=2.0 ** -6, grad_mode=GRAD_DYADIC,
                        w0_mode=W0_PHILOX, F=2)
        assert explore(cfg)[0] == n == {0: 200, 1: 252}[D]


def test_pins_catch_plausible_mistakes(monkeypatch):
    """The brute-force pin fails for plausible oracle bugs: an off-by-one gate
    (D+1 instead of D), and a wave aggregate that drops its first minibatch."""
    orig_gate = WSPOracle.gate_open

    def loose_gate(self, v):
        ok, pull = orig_gate(self, v)
        return (self.c_local[v] - self.c_global <= self.cfg.D + 1), pull

    monkeypatch.setattr(WSPOracle, "gate_open", loose_gate)
    with pytest.raises(AssertionError):
        n, _ = explore(_cfg(2, 0))
        assert n == 70400
    monkeypatch.setattr(WSPOracle, "gate_open", orig_gate)

    orig_complete = WSPOracle.complete

    def dropping_complete(self, t, v, p):
        out = orig_complete(self, t, v, p)
        if (p - 1) % self.cfg.Nm == 0:
            self.acc[v] = np.zeros_like(self.acc[v])     # forgets u of the 1st minibatch
        return out

    monkeypatch.setattr(WSPOracle, "complete", dropping_complete)
    with pytest.raises(AssertionError):
        explore(_cfg(2, 1))


@pytest.mark.parametrize("D,expected", [(0, 200), (1, 252)])
def test_bruteforce_momentum_update_frequency(D, expected):
    """The momentum brute force with F = 2 (NEXT-4: one push per two waves,
    P:1086-1087): 2 VW x 2 clocks x 8 params, N_m = 1."""
    cfg = WSPConfig("bf", 2, 1, D, 8, 2, (1, 1), lr=2.0 ** -6, grad_mode=GRAD_DYADIC,
                    w0_mode=W0_PHILOX, F=2, momentum=0.5)
    n, stats = explore(cfg)
    assert n == expected and stats["starts"] > 0


def test_momentum_pin_catches_plausible_mistake(monkeypatch):
    """The momentum brute force fails when the PS applies the previous m
    before updating it (w += m; m = mu m + u~), a plausible heavy-ball slip."""
    from oracle.wsp import F32

    def stale_push(self, t, v, c):
        ut = self.acc[v]
        self.wg = self.wg + self.m
        self.m = (F32(self.cfg.momentum) * self.m) + ut
        self.commit.append((v, c))
        self.c_local[v] = c + 1
        self.c_global = min(self.c_local)
        self.acc_count[v] = 0

    monkeypatch.setattr(WSPOracle, "push", stale_push)
    with pytest.raises(AssertionError):
        explore(_cfg(1, 0, momentum=0.5))


@pytest.mark.parametrize("Nm,D,W", [(1, 0, 3), (1, 1, 3), (2, 0, 3), (2, 1, 4), (3, 0, 3)])
def test_global_staleness_bound_is_tight(Nm, D, W):
    """P4: minibatch p is guaranteed every global update of
    minibatches 1..p-(s_global+1), s_global = (D+2) N_m - 2. Over every
    interleaving, the oldest other-VW state any START(p) can hold never goes
    below that floor, and the floor is attained: some START reads exactly it
    (the paper's example, minibatch 11 needs only 1..4 at N_m = 4, D = 0)."""
    from oracle import version_floor
    seen = {}
    cfg = WSPConfig("bf", 2, Nm, D, 8, W, (1, 1), lr=2.0 ** -6,
                    grad_mode=GRAD_DYADIC, w0_mode=W0_PHILOX)
    explore(cfg, seen)
    attained = 0
    for (v, p), top in seen.items():
        fl = max(0, version_floor(p, Nm, D))
        assert top >= fl, (v, p, top, fl)
        if fl > 0 and fl % Nm == 0:          # the floor ends a wave: reached exactly
            assert top == fl, (v, p, top, fl)
            attained += 1
    assert attained > 0


@pytest.mark.parametrize("Nm,D,W", [(1, 0, 3), (1, 1, 3), (2, 0, 3), (2, 1, 4), (1, 2, 5)])
def test_clock_distance_bound_is_tight(Nm, D, W):
    """P11 (north_star "no VW's clock runs more than D+1 waves past the
    slowest"): over every interleaving the clock distance never exceeds D+1,
    and some interleaving reaches D+1 (a fast VW that has pushed its gated
    wave while the slow one has pushed none beyond c_global)."""
    cfg = WSPConfig("bf", 2, Nm, D, 8, W, (1, 1), lr=2.0 ** -6,
                    grad_mode=GRAD_DYADIC, w0_mode=W0_PHILOX)
    _, stats = explore(cfg)
    assert stats["max_gap"] == D + 1

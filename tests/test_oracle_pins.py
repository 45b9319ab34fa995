"""Pins of the CPU oracle against what the paper and the mathematics fix
(no GPU). Each test names the pin and the passage."""
import os
import random

import numpy as np
import pytest

from oracle import (gradient, initial_weights, philox4x32_10, run_schedule,
                    s_global, version_floor, wave_range)
from oracle.wsp import WSPOracle, update, wave_of
from workloads import (C1, C1_SKEW, C2, C3, GRAD_DYADIC, GRAD_FLOAT, LOCAL_AT_LEAST,
                       LOCAL_STRICT, PULL_EAGER, PULL_LAZY, TAU_NP, W0_PHILOX,
                       W0_ZERO, WSPConfig)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                rows.append(line.split())
    return rows


# ----------------------------------------------------------------------------- P14
def test_philox_known_answers():
    for row in _golden("philox_kat.txt"):
        vals = [int(x, 16) for x in row]
        out = philox4x32_10(*vals[:4], vals[4], vals[5])
        assert [int(w) for w in out] == vals[6:10]


def test_philox_vectorised_matches_scalar():
    blk = np.arange(37, dtype=np.uint64) * np.uint64(2654435761)
    vec = philox4x32_10(blk, 3, 5, 0, 123, 456)
    for j in range(0, 37, 5):
        sc = philox4x32_10(int(blk[j]), 3, 5, 0, 123, 456)
        assert [int(w[j]) for w in vec] == [int(s) for s in sc]


# ----------------------------------------------------------------------------- P1-P3
def test_paper_worked_examples():
    for row in _golden("paper_examples.txt"):
        kind, args = row[0], [int(x) for x in row[1:]]
        if kind == "wave_range":
            c, Nm, lo, hi = args
            assert wave_range(c, Nm) == (lo, hi)
        elif kind == "s_global":
            s_local, D, val = args
            assert s_global(s_local + 1, D) == val
        elif kind == "version_floor":
            p, s_local, D, val = args
            assert version_floor(p, s_local + 1, D) == val
        elif kind == "gate":
            c_local, c_global, D, ok = args
            cfg = C1.replace(D=D)
            sm = WSPOracle(cfg, np.arange(4))
            sm.c_local = [c_local, c_global]
            sm.c_global = c_global
            assert sm.gate_open(0)[0] == bool(ok)
        else:
            raise AssertionError(kind)


def test_clock_advances_only_after_all_pushed():
    """c_global 0 -> 1 only after both VWs push wave 0."""
    r = run_schedule(C1_SKEW)
    pushes = [ln.split() for ln in r.trace if ln.split()[3] == "PUSH"]
    assert pushes[0][2] == "0" and pushes[0][7] == "0"        # vw0 pushed, c_global 0
    assert pushes[1][2] == "1" and pushes[1][7] == "1"        # vw1 pushed, c_global 1


def test_d0_narrative_minibatch_8():
    """with D=0, N_m=4 the VW pushes after minibatch 4, waits before
    minibatch 8, while 5, 6 and 7 have already started."""
    cfg = WSPConfig("nar", 2, 4, 0, 64, 3, (100, 170))
    r = run_schedule(cfg)
    ev = [ln.split() for ln in r.trace if ln.split()[2] == "0"]
    kinds = [(e[3], int(e[4])) for e in ev]
    i_push = kinds.index(("PUSH", 4))
    i_block = kinds.index(("BLOCK", 8))
    i_start8 = kinds.index(("START", 8))
    for q in (5, 6, 7):
        assert kinds.index(("START", q)) < i_push
    assert i_push < i_block < i_start8
    t_start8 = int(ev[i_start8][0])
    t_other_push = min(int(ln.split()[0]) for ln in r.trace
                       if ln.split()[2] == "1" and ln.split()[3] == "PUSH")
    assert t_start8 == t_other_push


def test_first_minibatches_see_w0():
    """P5 / P:835-836: w_1 = ... = w_{s_local+1} = w_0."""
    cfg = C2.replace(nparams=256, waves=3)
    r = run_schedule(cfg, record_snapshots=True)
    w0 = initial_weights(np.arange(256), cfg)
    for t, v, p, snap in r.snapshots:
        if p <= cfg.Nm:
            assert np.array_equal(snap, w0)


# ----------------------------------------------------------------------------- P8
def _exact_sum_u(idx, cfg, pairs):
    tot = np.zeros(idx.size, dtype=np.float64)
    for v, p in pairs:
        tot += -float(np.float32(cfg.lr)) * gradient(idx, v, p, cfg).astype(np.float64)
    return tot


def test_bsp_limit_dyadic_exact():
    """P8: N_m=1 (naive MP), D=0 (BSP-like) is synchronous
    data-parallel SGD: w_final = w0 - lr * sum of all gradients, exactly."""
    cfg = C1.replace(waves=12, w0_mode=W0_PHILOX)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg, record_snapshots=True)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    allp = [(v, p) for v in range(cfg.num_vw) for p in range(1, cfg.waves + 1)]
    expect = w0 + _exact_sum_u(idx, cfg, allp)
    assert np.array_equal(r.wg.astype(np.float64), expect)
    # every START(p) snapshot = w0 + all VWs' updates of minibatches < p
    for t, v, p, snap in r.snapshots:
        pairs = [(vv, q) for vv in range(cfg.num_vw) for q in range(1, p)]
        assert np.array_equal(snap.astype(np.float64), w0 + _exact_sum_u(idx, cfg, pairs))


def test_bsp_limit_float_within_rounding_bound():
    """P8 in FLOAT mode: the fp32 result is the exact sum to within the standard
    recursive-summation bound n * u * sum |terms| (Higham, Accuracy and Stability,
    eq. 4.4), with u = 2^-24 and per-term rounding of fl(-lr*g) included."""
    cfg = C1.replace(grad_mode=GRAD_FLOAT, lr=0.01, w0_mode=W0_PHILOX, waves=16,
                     nparams=1024)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    lr = 0.01                                  # the REAL lr, not fl32(lr)
    exact = w0.copy()
    absum = np.abs(w0).copy()
    for v in range(cfg.num_vw):
        for p in range(1, cfg.waves + 1):
            term = -lr * gradient(idx, v, p, cfg).astype(np.float64)
            exact += term
            absum += np.abs(term)
    n = cfg.num_vw * cfg.waves + 2
    bound = n * 2.0 ** -24 * absum + 2.0 ** -24 * np.abs(exact)
    assert np.all(np.abs(r.wg.astype(np.float64) - exact) <= bound)


# ----------------------------------------------------------------------------- P9-P12
def _rand_cfg(rng, **kw):
    N = rng.randint(1, 4)
    Nm = rng.randint(1, 4)
    D = rng.randint(0, 3)
    W = rng.randint(1, 6)
    tau = tuple(rng.randint(1, 9) for _ in range(N))
    base = dict(name="rand", num_vw=N, Nm=Nm, D=D, nparams=40, waves=W, tau=tau,
                lr=2.0 ** -6, grad_mode=GRAD_DYADIC, w0_mode=W0_PHILOX,
                pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
                local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]),
                lat=tuple(t * rng.randint(1, Nm + 1) for t in tau),
                seed=rng.randint(0, 2 ** 63))
    base.update(kw)
    return WSPConfig(**base)


def _version_sum(idx, cfg, v, a_v, commit_prefix, w0):
    """Declarative START snapshot: w0 + every pushed wave of the OTHER VWs in the
    held commit prefix + own updates 1..a_v (exact in DYADIC mode)."""
    pairs = [(v, q) for q in range(1, a_v + 1)]
    for (vv, c) in commit_prefix:
        if vv != v:
            lo, hi = wave_range(c, cfg.Nm)
            pairs += [(vv, q) for q in range(lo, hi + 1)]
    return w0 + _exact_sum_u(idx, cfg, pairs)


@pytest.mark.parametrize("seed", range(40))
def test_random_configs_invariants(seed):
    """P9 conservation, P11 clock bound, P12 read bound, P4 version floor, and the
    START snapshot = declarative version-set sum, on random configs (DYADIC)."""
    rng = random.Random(seed)
    cfg = _rand_cfg(rng)
    idx = np.arange(cfg.nparams)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    admissions = []

    def on_tick(t, sm):
        admissions.append((list(sm.c_local), sm.c_global))

    r = run_schedule(cfg, record_snapshots=True, on_tick=on_tick)
    # P9: w_global = w0 + sum of every update, exactly
    allp = [(v, p) for v in range(cfg.num_vw) for p in range(1, cfg.waves * cfg.Nm + 1)]
    assert np.array_equal(r.wg.astype(np.float64), w0 + _exact_sum_u(idx, cfg, allp))
    assert len(r.commit) == cfg.num_vw * cfg.waves
    # P11: the clock distance never exceeds D+1 (north_star), admissions obey D
    assert r.max_clock_gap <= cfg.D + 1
    for ln in r.trace:
        f = ln.split()
        if f[3] in ("PULL", "ADMIT"):
            assert int(f[6]) - int(f[7]) <= cfg.D or cfg.pull_policy == PULL_LAZY
    # P12 (STRICT exact) / AT_LEAST lower bound, and P4 version floor
    for (v, p, a_v, held_K) in r.start_versions:
        if cfg.local_semantics == LOCAL_STRICT:
            assert a_v == max(0, p - cfg.Nm)
        else:
            assert a_v >= max(0, p - cfg.Nm)
        f = version_floor(p, cfg.Nm, cfg.D)
        if f > 0:
            need = wave_of(f, cfg.Nm)
            have = set(r.commit[:held_K])
            for vv in range(cfg.num_vw):
                if vv != v:
                    assert all((vv, c) in have for c in range(need + 1)), (v, p, f)
            assert a_v >= f
    # snapshot of every START = declarative version-set sum
    for (t, v, p, snap), (v2, p2, a_v, held_K) in zip(r.snapshots, r.start_versions):
        assert (v, p) == (v2, p2)
        expect = _version_sum(idx, cfg, v, a_v, r.commit[:held_K], w0)
        assert np.array_equal(snap.astype(np.float64), expect), (v, p)
    # final w_local: every due fold applied, no final pull (Z16)
    for v in range(cfg.num_vw):
        last_pull = [ln.split() for ln in r.trace
                     if ln.split()[2] == str(v) and ln.split()[3] == "PULL"]
        held_K = int(last_pull[-1][10]) if last_pull else 0
        a_v = cfg.waves * cfg.Nm
        expect = _version_sum(idx, cfg, v, a_v, r.commit[:held_K], w0)
        assert np.array_equal(r.wl[v].astype(np.float64), expect)


def _abs_sum_u(idx, cfg, pairs):
    tot = np.zeros(idx.size, dtype=np.float64)
    for v, p in pairs:
        tot += np.abs(float(np.float32(cfg.lr)) * gradient(idx, v, p, cfg).astype(np.float64))
    return tot


def _version_pairs(cfg, v, a_v, commit_prefix):
    pairs = [(v, q) for q in range(1, a_v + 1)]
    for (vv, c) in commit_prefix:
        if vv != v:
            lo, hi = wave_range(c, cfg.Nm)
            pairs += [(vv, q) for q in range(lo, hi + 1)]
    return pairs


def _within_summation_bound(got, w0, idx, cfg, pairs):
    """|fl32 result - exact| <= gamma_n * (|w0| + sum|u|) + per-term rounding:
    Higham, Accuracy and Stability, eq. 4.4 (any summation order, n terms,
    gamma_n = n u / (1 - n u), u = 2^-24), plus u |term| for fl(-lr * g)."""
    exact = w0 + _exact_sum_u(idx, cfg, pairs)
    absum = np.abs(w0) + _abs_sum_u(idx, cfg, pairs)
    n = len(pairs) + 1
    u = 2.0 ** -24
    bound = (n * u / (1 - n * u) + u) * absum
    return bool(np.all(np.abs(got.astype(np.float64) - exact) <= bound))


@pytest.mark.parametrize("seed", list(range(24)) + ["np", "hd"])
def test_float_snapshots_within_summation_bound(seed):
    """FLOAT mode, D > 0, heterogeneous speeds (the case whose exact bits only
    the oracle fixes): every START snapshot, the final
    w_global and every final w_local hold the values of their version
    set (the same sets the DYADIC pins fix exactly) to within the recursive
    summation bound of Higham eq. 4.4; a snapshot with one update dropped or
    with one extra update does not."""
    if seed in ("np", "hd"):             # C2's NP speeds at D = 1; C3's HD speeds, D = 4
        cfg = (C2.replace(D=1) if seed == "np" else C3).replace(
            nparams=64, waves=6, lr=0.01, grad_mode=GRAD_FLOAT, w0_mode=W0_PHILOX)
    else:
        rng = random.Random(1000 + seed)
        cfg = _rand_cfg(rng, grad_mode=GRAD_FLOAT, lr=0.01, D=rng.randint(1, 4),
                        nparams=64)
    idx = np.arange(cfg.nparams)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    r = run_schedule(cfg, record_snapshots=True)
    allp = [(v, p) for v in range(cfg.num_vw) for p in range(1, cfg.waves * cfg.Nm + 1)]
    assert _within_summation_bound(r.wg, w0, idx, cfg, allp)
    checked_neg = 0
    for (t, v, p, snap), (v2, p2, a_v, held_K) in zip(r.snapshots, r.start_versions):
        assert (v, p) == (v2, p2)
        pairs = _version_pairs(cfg, v, a_v, r.commit[:held_K])
        assert _within_summation_bound(snap, w0, idx, cfg, pairs), (v, p)
        if pairs:                                   # a dropped update is caught
            assert not _within_summation_bound(snap, w0, idx, cfg, pairs[1:])
            checked_neg += 1
        missing = [q for q in allp if q not in pairs]
        if missing:                                 # so is an extra one
            assert not _within_summation_bound(snap, w0, idx, cfg, pairs + missing[:1])
    for v in range(cfg.num_vw):
        last_pull = [ln.split() for ln in r.trace
                     if ln.split()[2] == str(v) and ln.split()[3] == "PULL"]
        held_K = int(last_pull[-1][10]) if last_pull else 0
        pairs = _version_pairs(cfg, v, cfg.waves * cfg.Nm, r.commit[:held_K])
        assert _within_summation_bound(r.wl[v], w0, idx, cfg, pairs)
    assert checked_neg > 0 or cfg.waves * cfg.Nm <= cfg.Nm


def test_d0_lockstep():
    """P6: with D=0 every admission sees all local clocks equal."""
    for tau in (TAU_NP, (100, 173, 260), (5, 7)):
        cfg = WSPConfig("ls", len(tau), 3, 0, 16, 8, tau, lr=2.0 ** -6,
                        grad_mode=GRAD_DYADIC)
        r = run_schedule(cfg)
        for ln in r.trace:
            f = ln.split()
            if f[3] == "PULL":
                # c_local of the admitted VW equals c_global = min; no VW is ahead
                # by more than the one pushed wave it is waiting on
                assert int(f[6]) == int(f[7])
        assert r.max_clock_gap <= 1


def test_wait_non_increasing_in_D():
    """P7 (P:343-345 wait(D=4) = 62% of wait(D=0)): total wait ticks do
    not increase with D for fixed speeds."""
    for tau, Nm in ((TAU_NP, 4), ((250, 250, 330, 330, 346, 346, 421, 421), 8),
                    ((3, 5, 7), 2), ((100, 173), 1)):
        waits = []
        for D in range(0, 6):
            cfg = WSPConfig("w", len(tau), Nm, D, 4, 24, tau, lr=2.0 ** -6,
                            grad_mode=GRAD_DYADIC)
            waits.append(sum(run_schedule(cfg).wait))
        assert all(a >= b for a, b in zip(waits, waits[1:])), waits


def test_single_vw_and_unbounded_D():
    """P10: N=1 never blocks and EAGER keeps w_local = w_global after each pull;
    D >= W-1 with LAZY never pulls and w_local = w0 + own updates only."""
    cfg = WSPConfig("one", 1, 3, 0, 32, 6, (7,), lr=2.0 ** -6, grad_mode=GRAD_DYADIC)
    r = run_schedule(cfg)
    assert r.wait == [0] and not any("BLOCK" in ln for ln in r.trace)
    cfg2 = WSPConfig("lazy", 3, 2, 5, 32, 6, (3, 5, 8), lr=2.0 ** -6,
                     grad_mode=GRAD_DYADIC, pull_policy=PULL_LAZY)
    r2 = run_schedule(cfg2)
    assert r2.pulls == [0, 0, 0]
    idx = np.arange(32)
    w0 = initial_weights(idx, cfg2).astype(np.float64)
    for v in range(3):
        own = [(v, p) for p in range(1, 13)]
        assert np.array_equal(r2.wl[v].astype(np.float64), w0 + _exact_sum_u(idx, cfg2, own))


# ----------------------------------------------------------------------------- P15
def test_momentum_zero_is_sgd_bitwise():
    cfg = C2.replace(nparams=512, waves=5, D=1)
    a = run_schedule(cfg)
    b = run_schedule(cfg.replace(momentum=1e-30))      # forces the momentum branch
    assert a.trace == b.trace
    c = run_schedule(cfg.replace(momentum=0.0))
    assert np.array_equal(a.wg, c.wg)


def test_momentum_heavy_ball_closed_form():
    """P15 (Z11): heavy ball m_k = mu m_{k-1} + u~_k, w_K = w0 + sum_k m_k, whose
    closed form is w_K = w0 + sum_j u~_j (1 - mu^(K-j+1)) / (1 - mu). Checked in
    fp64 against the fp32 oracle with a rounding-error bound."""
    mu = 0.9
    cfg = WSPConfig("mom", 1, 1, 0, 256, 40, (10,), lr=0.01, momentum=mu,
                    grad_mode=GRAD_FLOAT, w0_mode=W0_PHILOX)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg)
    K = cfg.waves
    w = initial_weights(idx, cfg).astype(np.float64)
    mag = np.abs(w).copy()
    for j in range(1, K + 1):
        u = update(idx, 0, j, cfg).astype(np.float64)
        w += u * (1 - mu ** (K - j + 1)) / (1 - mu)
        mag += np.abs(u) / (1 - mu)
    assert np.all(np.abs(r.wg.astype(np.float64) - w) <= 4 * K * 2.0 ** -24 * mag + 1e-12)


def _heavy_ball_snapshot(idx, cfg, v, a_v, prefix, w0, mu):
    """w0 + sum_j u~_(j) (1 - mu^(K-j+1)) / (1 - mu) over the commit prefix
    (K = its length; Z11 heavy ball applied in commit order) + the
    VW's own updates not in a pushed wave of the prefix, up to a_v (P:838-839,
    "w_local = w_global + not-yet-pushed local updates"); fp64 from the fp32
    terms u_p. Returns (value, magnitude for the rounding bound)."""
    K = len(prefix)
    w = w0.copy()
    mag = np.abs(w0).copy()
    own_pushed = set()
    for j, (vv, c) in enumerate(prefix, start=1):
        lo, hi = wave_range(c, cfg.Nm)
        ut = np.zeros_like(w0)
        for q in range(lo, hi + 1):
            ut += update(idx, vv, q, cfg).astype(np.float64)
        w += ut * (1 - mu ** (K - j + 1)) / (1 - mu)
        mag += np.abs(ut) / (1 - mu)
        if vv == v:
            own_pushed.update(range(lo, hi + 1))
    for q in range(1, a_v + 1):
        if q not in own_pushed:
            u = update(idx, v, q, cfg).astype(np.float64)
            w += u
            mag += np.abs(u)
    return w, mag


@pytest.mark.parametrize("seed", list(range(16)) + ["np"])
def test_momentum_snapshots_heavy_ball_closed_form(seed):
    """P15 with several VWs, D > 0 and heterogeneous speeds: every START
    snapshot and the final w_global equal the heavy-ball closed form over the
    commit order (Z11) plus the VW's own unpushed updates, in fp64 within a
    rounding bound; the same snapshot with plain-SGD weights (mu dropped) or
    with one pushed wave missing does not."""
    mu = 0.9
    if seed == "np":                     # C2's NP speeds, EAGER / STRICT, D = 1
        cfg = C2.replace(nparams=64, waves=5, D=1, lr=0.01, momentum=mu,
                         grad_mode=GRAD_FLOAT, w0_mode=W0_PHILOX)
    else:
        rng = random.Random(2000 + seed)
        cfg = _rand_cfg(rng, grad_mode=GRAD_FLOAT, lr=0.01, momentum=mu,
                        D=rng.randint(1, 3), nparams=64)
    idx = np.arange(cfg.nparams)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    r = run_schedule(cfg, record_snapshots=True)
    n = cfg.num_vw * cfg.waves * cfg.Nm + cfg.num_vw * cfg.waves + 2
    tol = lambda mag: 4 * n * 2.0 ** -24 * mag
    w, mag = _heavy_ball_snapshot(idx, cfg, -1, 0, r.commit, w0, mu)
    assert np.all(np.abs(r.wg.astype(np.float64) - w) <= tol(mag))
    negatives = 0
    for (t, v, p, snap), (v2, p2, a_v, held_K) in zip(r.snapshots, r.start_versions):
        assert (v, p) == (v2, p2)
        prefix = r.commit[:held_K]
        w, mag = _heavy_ball_snapshot(idx, cfg, v, a_v, prefix, w0, mu)
        err = np.abs(snap.astype(np.float64) - w)
        assert np.all(err <= tol(mag)), (v, p)
        if any(vv != v for vv, _ in prefix):
            sgd = _version_sum(idx, cfg, v, a_v, prefix, w0)
            if held_K >= 2:                      # mu matters once two pushes stack
                assert not np.all(np.abs(snap.astype(np.float64) - sgd) <= tol(mag))
            k = next(j for j, (vv, _) in enumerate(prefix) if vv != v)
            w_drop, _ = _heavy_ball_snapshot(idx, cfg, v, a_v,
                                             prefix[:k] + prefix[k + 1:], w0, mu)
            assert not np.all(np.abs(snap.astype(np.float64) - w_drop) <= tol(mag))
            negatives += 1
    if seed == "np":
        assert negatives > 0


# ----------------------------------------------------------------------------- P16
def test_determinism_and_sampling():
    cfg = C2.replace(nparams=3000, waves=4, D=1)
    a = run_schedule(cfg)
    b = run_schedule(cfg)
    assert a.trace == b.trace and np.array_equal(a.wg, b.wg)
    idx = np.array([0, 1, 2, 3, 17, 1023, 1024, 2047, 2999])
    s = run_schedule(cfg, idx=idx)
    assert s.trace == a.trace
    assert np.array_equal(s.wg, a.wg[idx])
    for v in range(cfg.num_vw):
        assert np.array_equal(s.wl[v], a.wl[v][idx])


def test_gradient_modes():
    idx = np.arange(4096)
    g = gradient(idx, 1, 3, C2)
    assert g.dtype == np.float32 and g.min() >= -0.5 and g.max() < 0.5
    assert abs(float(g.mean())) < 0.02
    gd = gradient(idx, 1, 3, C1)
    assert set(np.unique(gd).tolist()) <= set(range(-8, 8))
    w0 = initial_weights(idx, C2)
    assert w0.min() >= -1 and w0.max() < 1


def test_spec_timeline_examples():
    """SPEC.md's timeline examples, in the tick model (Nm = 1, so a
    wave is one minibatch and L = tau): homogeneous speeds never wait; wave
    durations {1, 2} at D = 0 make the fast VW wait one unit per clock --
    it pushes at t = c*100 + 100 and is admitted when the slow VW's push of the
    same clock arrives, 100 ticks later, for every clock but the last (no gated
    START remains, Z16) -- and D = 4 waits strictly less."""
    for tau in ((100, 100), (50, 50, 50)):
        r = run_schedule(WSPConfig("h", len(tau), 1, 0, 8, 8, tau, lr=2.0 ** -6,
                                   grad_mode=GRAD_DYADIC))
        assert r.wait == [0] * len(tau)
    W = 8
    base = WSPConfig("t", 2, 1, 0, 8, W, (100, 200), lr=2.0 ** -6, grad_mode=GRAD_DYADIC)
    r0 = run_schedule(base)
    assert r0.wait == [(W - 1) * 100, 0]
    r4 = run_schedule(base.replace(D=4))
    assert r4.wait[0] < r0.wait[0] and r4.wait[1] == 0

"""Pins of the oracle's weight-dependent workload and of
the paper's convergence-analysis decomposition (section 6,
P:1497-1521) on the version sets of the trace. CPU only.

With g = a (w_p - b) + sigma xi the updates depend on the weights each
minibatch read at its START, so staleness becomes numerically observable:
  * BSP limit (Nm = 1, D = 0, sigma = 0, equal speeds): every VW reads w_p with
    all N VWs' updates of minibatches < p, so
    w - b = (1 - N lr a)^W (w0 - b)  (gradient descent on a/2 ||w - b||^2);
  * one VW with Nm in flight: minibatch p reads exactly its own updates up to
    p - Nm (north_star) -- the delayed recurrence
    e_p = e_{p-1} - lr a e_{p-Nm} (e = w - b, sigma = 0), e_1..e_Nm = e_0;
  * any config: every START snapshot = w0 + the sum of the updates in its
    version set (own 1..a_v, the other VWs' pushed waves of the held commit
    prefix), the updates recomputed from the snapshots they read.
The decomposition of section 6 (the "noisy weight" w~_{n,p} = w0 + all
updates of minibatches <= p - s_g - 1 + own updates in C ⊆ [p - s_g, p - 1]
+ other workers' updates in E ⊆ [p - s_g, p + s_g + s_l], s_g = s_global,
s_l = s_local + 1) and Lemma 1's count bound are checked on every START.
"""
import random

import numpy as np
import pytest

from oracle import convex_target, initial_weights, run_schedule, s_global, version_floor
from oracle.wsp import update, wave_of, wave_range
from workloads import (GRAD_CONVEX, GRAD_DYADIC, LOCAL_AT_LEAST, LOCAL_STRICT, PULL_EAGER,
                       PULL_LAZY, W0_PHILOX, WSPConfig)


def convex_cfg(**kw):
    base = dict(name="cvx", num_vw=2, Nm=1, D=0, nparams=257, waves=16, tau=(7, 7),
                lr=0.05, grad_mode=GRAD_CONVEX, w0_mode=W0_PHILOX, conv_a=0.5, conv_sigma=0.0)
    base.update(kw)
    return WSPConfig(**base)


def normwise(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("N", [1, 2, 4])
def test_convex_bsp_closed_form(N):
    cfg = convex_cfg(num_vw=N, tau=(7,) * N)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg)
    e0 = initial_weights(idx, cfg).astype(np.float64) - convex_target(idx, cfg)
    k = 1.0 - N * cfg.lr * cfg.conv_a
    want = k ** cfg.waves * e0
    got = r.wg.astype(np.float64) - convex_target(idx, cfg)
    # 16 steps of a contraction: a few float32 roundings per step
    assert normwise(got, want) < 1e-5
    # w_local: no final pull (Z16) -- the last wave adds only its own update
    want_l = (1.0 - cfg.lr * cfg.conv_a) * k ** (cfg.waves - 1) * e0
    for v in range(N):
        assert normwise(r.wl[v].astype(np.float64) - convex_target(idx, cfg), want_l) < 1e-5


@pytest.mark.parametrize("Nm,D,policy", [(2, 0, PULL_EAGER), (3, 1, PULL_EAGER),
                                          (4, 3, PULL_LAZY), (5, 0, PULL_LAZY)])
def test_convex_single_vw_delayed_recurrence(Nm, D, policy):
    """One VW: START(p) sees its own updates up to exactly p - Nm."""
    cfg = convex_cfg(num_vw=1, Nm=Nm, D=D, tau=(5,), waves=8, pull_policy=policy)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg, record_snapshots=True)
    b = convex_target(idx, cfg).astype(np.float64)
    e = {0: initial_weights(idx, cfg).astype(np.float64) - b}
    kappa = cfg.lr * cfg.conv_a
    P = cfg.waves * Nm
    for p in range(1, P + 1):
        e[p] = e[0] if p <= Nm else e[p - 1] - kappa * e[p - Nm]
    for (t, v, p, snap) in r.snapshots:
        assert normwise(snap.astype(np.float64) - b, e[p]) < 1e-5, p
    # the final w_local holds every update 1..P (u_q = -lr a e_q): minibatch P's
    # weights plus the Nm updates P-Nm+1..P it did not see
    fin = e[P] - kappa * sum(e[q] for q in range(P - Nm + 1, P + 1))
    assert normwise(r.wl[0].astype(np.float64) - b, fin) < 1e-5


def _rand_cfg(rng, **kw):
    N = rng.randint(1, 4)
    Nm = rng.randint(1, 4)
    tau = tuple(rng.randint(1, 9) for _ in range(N))
    base = dict(name="rc", num_vw=N, Nm=Nm, D=rng.randint(0, 3), nparams=40,
                waves=rng.randint(1, 6), tau=tau, lr=0.05,
                pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
                local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]),
                lat=tuple(t * rng.randint(1, Nm + 1) for t in tau),
                seed=rng.randint(0, 2 ** 63), grad_mode=GRAD_CONVEX, conv_sigma=0.5)
    base.update(kw)
    return WSPConfig(**base)


@pytest.mark.parametrize("seed", range(30))
def test_convex_snapshots_are_version_set_sums(seed):
    rng = random.Random(seed)
    cfg = _rand_cfg(rng)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg, record_snapshots=True)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    snap = {(v, p): s for (t, v, p, s) in r.snapshots}
    # each update recomputed from the weights its minibatch read at START
    u = {k: update(idx, k[0], k[1], cfg, w).astype(np.float64) for k, w in snap.items()}
    for (t, v, p, s), (v2, p2, a_v, held_K) in zip(r.snapshots, r.start_versions):
        pairs = [(v, q) for q in range(1, a_v + 1)]
        for (vv, c) in r.commit[:held_K]:
            if vv != v:
                lo, hi = wave_range(c, cfg.Nm)
                pairs += [(vv, q) for q in range(lo, hi + 1)]
        want = w0 + sum((u[k] for k in pairs), np.zeros_like(w0))
        assert normwise(s, want) < 1e-5, (v, p)
    # conservation with weight-dependent updates: w_global = w0 + every update
    allu = sum(u.values(), np.zeros_like(w0))
    assert normwise(r.wg, w0 + allu) < 1e-5


@pytest.mark.parametrize("seed", range(40))
def test_lemma1_decomposition_on_version_sets(seed):
    """Section 6: w~_{n,p} contains every update of minibatches
    <= p - s_g - 1 of every worker, own extras C ⊆ [p - s_g, p - 1] and other
    workers' extras E ⊆ [p - s_g, p + s_g + s_l] x ([1,N] minus n); Lemma 1
    (P:1531): |R| + |Q| <= |E| <= (2 s_g + s_l)(N - 1)."""
    rng = random.Random(seed)
    cfg = _rand_cfg(rng, grad_mode=GRAD_DYADIC, lr=2.0 ** -6)
    r = run_schedule(cfg)
    sg, sl = s_global(cfg.Nm, cfg.D), cfg.Nm
    for (v, p, a_v, held_K) in r.start_versions:
        own = set(range(1, a_v + 1))
        other = {}
        for (vv, c) in r.commit[:held_K]:
            if vv != v:
                lo, hi = wave_range(c, cfg.Nm)
                other.setdefault(vv, set()).update(range(lo, hi + 1))
        floor = version_floor(p, cfg.Nm, cfg.D)           # p - s_g - 1
        assert own >= set(range(1, floor + 1))
        assert all(p - sg <= q <= p - 1 for q in own - set(range(1, floor + 1)))
        E = 0
        for vv in range(cfg.num_vw):
            if vv == v:
                continue
            got = other.get(vv, set())
            assert got >= set(range(1, floor + 1)), (v, p, vv)
            extra = got - set(range(1, floor + 1))
            assert all(p - sg <= q <= p + sg + sl for q in extra), (v, p, vv, sorted(extra))
            E += len(extra)
        assert E <= (2 * sg + sl) * (cfg.num_vw - 1), (v, p, E)

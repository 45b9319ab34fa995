"""Pins of the update frequency factor F (a drafted
variant of the paper): the clock unit becomes F waves -- a VW
with clock c aggregates minibatches c F (s_local+1) + 1 .. (c+1) F (s_local+1)
and pushes once, keeps executing up to (F-1)(s_local+1) +
s_local further minibatches on its last synchronised weights,
and s_global = F (D+2)(s_local+1) - 2. CPU only."""
import random

import numpy as np
import pytest

from oracle import initial_weights, run_schedule, s_global, version_floor
from oracle.wsp import clock_range, update
from workloads import (GRAD_DYADIC, LOCAL_AT_LEAST, LOCAL_STRICT, PULL_EAGER, PULL_LAZY,
                       W0_PHILOX, WSPConfig)


def test_s_global_two_forms():
    # P:1090 prints both: F(D+2)(s_local+1) - 2 = F(D+1)(s_local+1) + (F-1)(s_local+1) + s_local - 1
    for F in range(1, 6):
        for D in range(0, 6):
            for Nm in range(1, 7):
                assert s_global(Nm, D, F) == F * (D + 2) * Nm - 2
    assert s_global(4, 0, 1) == 6 and s_global(4, 4, 1) == 22      # P:999 (F = 1)


def rand_cfg(rng, **kw):
    N = rng.randint(1, 4)
    Nm = rng.randint(1, 3)
    tau = tuple(rng.randint(1, 9) for _ in range(N))
    base = dict(name="f", num_vw=N, Nm=Nm, D=rng.randint(0, 2), nparams=24,
                waves=rng.randint(1, 4), tau=tau, lr=2.0 ** -6, grad_mode=GRAD_DYADIC,
                w0_mode=W0_PHILOX, pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
                local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]),
                lat=tuple(t * rng.randint(1, Nm + 1) for t in tau),
                seed=rng.randint(0, 2 ** 63), F=rng.randint(2, 4))
    base.update(kw)
    return WSPConfig(**base)


def exact_sum(idx, cfg, pairs):
    tot = np.zeros(idx.size, dtype=np.float64)
    for v, p in pairs:
        tot += update(idx, v, p, cfg).astype(np.float64)
    return tot


@pytest.mark.parametrize("seed", range(40))
def test_update_frequency_invariants(seed):
    rng = random.Random(seed)
    cfg = rand_cfg(rng)
    U = cfg.F * cfg.Nm
    idx = np.arange(cfg.nparams)
    w0 = initial_weights(idx, cfg).astype(np.float64)
    r = run_schedule(cfg, record_snapshots=True)
    P = cfg.waves * U
    # one push per clock, each the aggregate of U minibatches; conservation
    assert len(r.commit) == cfg.num_vw * cfg.waves
    allp = [(v, p) for v in range(cfg.num_vw) for p in range(1, P + 1)]
    assert np.array_equal(r.wg.astype(np.float64), w0 + exact_sum(idx, cfg, allp))
    assert r.max_clock_gap <= cfg.D + 1
    # gate events only guard the minibatches (c+2)*U
    for ln in r.trace:
        f = ln.split()
        if f[3] in ("BLOCK", "PULL", "ADMIT"):
            assert int(f[4]) % U == 0 and int(f[4]) >= 2 * U, ln
    for (t, v, p, snap), (v2, p2, a_v, held_K) in zip(r.snapshots, r.start_versions):
        if cfg.local_semantics == LOCAL_STRICT:
            assert a_v == max(0, p - cfg.Nm)                    # local staleness unchanged
        else:
            assert a_v >= max(0, p - cfg.Nm)
        have = set(r.commit[:held_K])
        fl = version_floor(p, cfg.Nm, cfg.D, cfg.F)          # s_global with F
        if fl > 0:
            need = (fl - 1) // U
            for vv in range(cfg.num_vw):
                if vv != v:
                    assert all((vv, c) in have for c in range(need + 1)), (v, p, fl)
            assert a_v >= fl
        pairs = [(v, q) for q in range(1, a_v + 1)]
        for (vv, c) in r.commit[:held_K]:
            if vv != v:
                lo, hi = clock_range(c, U)
                pairs += [(vv, q) for q in range(lo, hi + 1)]
        assert np.array_equal(snap.astype(np.float64), w0 + exact_sum(idx, cfg, pairs)), (v, p)


def test_f_pushes_less_often():
    """F = 2 halves the pushes of the same minibatches (the point of F)."""
    base = WSPConfig("f1", 2, 2, 0, 8, 8, (3, 4), lr=2.0 ** -6, grad_mode=GRAD_DYADIC)
    r1 = run_schedule(base)
    r2 = run_schedule(base.replace(F=2, waves=4))
    assert len(r1.commit) == 2 * len(r2.commit)
    assert np.array_equal(r1.wg, r2.wg)        # DYADIC: the same updates, exactly

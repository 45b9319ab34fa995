"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs. Same summation order on both sides, so the bar is
bit-exact fp32 weights (stronger than the north_star's 1e-5 relative) and
byte-identical clock/version traces."""
import os
import random
import tempfile

import numpy as np
import pytest

from oracle import gradient, run_schedule
from workloads import (C1, C1_SKEW, C2, C3, C4, C5, GRAD_CONVEX, GRAD_DYADIC, GRAD_EXTERNAL,
                       GRAD_FLOAT, LOCAL_AT_LEAST, LOCAL_STRICT, PULL_EAGER,
                       PULL_LAZY, W0_PHILOX, W0_ZERO, WSPConfig, sample_indices)

pytestmark = pytest.mark.gpu


class _HP:
    """The binding plus the library build under test (real CUDA library here;
    tests/test_engine_emu.py reuses these cases with the host emulation)."""

    def __init__(self, hetpipe, lib=None):
        self._m = hetpipe
        self.lib = lib

    def __getattr__(self, k):
        return getattr(self._m, k)

    def Context(self, cfg):
        return self._m.Context(cfg, lib=self.lib)


@pytest.fixture(scope="module")
def hp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2005_14038_b200 import build, hetpipe
    build.build()
    return _HP(hetpipe)


def run_device(hp, cfg, apply_mode=0, acc_slots=2, **over):
    ctx = hp.Context(hp.config_from(cfg, apply_mode=apply_mode, acc_slots=acc_slots, **over))
    ctx.run_schedule(cfg.tau, cfg.latency())
    with tempfile.NamedTemporaryFile(suffix=".trace") as f:
        trace = ctx.trace_lines(f.name)
    wg = ctx.read_weights(-1)
    wl = [ctx.read_weights(v) for v in range(cfg.num_vw)]
    m = ctx.read_weights(-2) if cfg.momentum else None
    st = ctx.stats()
    ctx.close()
    return trace, wg, wl, m, st


def assert_same(o, trace, wg, wl, idx=None):
    assert trace == o.trace
    sel = (lambda a: a) if idx is None else (lambda a: a[idx])
    assert np.array_equal(sel(wg), o.wg)
    for v, w in enumerate(wl):
        assert np.array_equal(sel(w), o.wl[v]), f"w_local({v})"


@pytest.mark.parametrize("cfg", [C1, C1_SKEW], ids=["C1", "C1-skew"])
@pytest.mark.parametrize("apply_mode", [0, 1])
def test_c1_bsp_limit_bit_exact(hp, cfg, apply_mode):
    o = run_schedule(cfg)
    trace, wg, wl, _, st = run_device(hp, cfg, apply_mode)
    assert_same(o, trace, wg, wl)
    assert st.commits == cfg.num_vw * cfg.waves == st.applied
    assert list(st.wait_ticks[:cfg.num_vw]) == o.wait
    assert list(st.pulls[:cfg.num_vw]) == o.pulls


def _rand_cfg(seed):
    rng = random.Random(seed)
    N = rng.randint(1, 5)
    Nm = rng.randint(1, 5)
    tau = tuple(rng.randint(1, 12) for _ in range(N))
    mode = rng.choice([GRAD_FLOAT, GRAD_DYADIC])
    return WSPConfig(
        "rand", N, Nm, rng.randint(0, 3), rng.choice([1, 3, 4, 61, 256, 1027, 4099]),
        rng.randint(1, 7), tau, lr=(0.01 if mode == GRAD_FLOAT else 2.0 ** -6),
        momentum=rng.choice([0.0, 0.0, 0.9]), seed=rng.randint(0, 2 ** 64 - 1),
        grad_mode=mode, w0_mode=rng.choice([W0_ZERO, W0_PHILOX]),
        pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
        local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]),
        lat=tuple(t * rng.randint(1, Nm + 1) for t in tau))


@pytest.mark.parametrize("seed", range(48))
def test_random_configs_bit_exact(hp, seed):
    """Random N, Nm, D, P (ragged tails), W, speeds, momentum, EAGER/LAZY,
    STRICT/AT_LEAST, apply modes and ring depths: identical traces and arrays."""
    cfg = _rand_cfg(seed)
    o = run_schedule(cfg)
    rng = random.Random(1000 + seed)
    trace, wg, wl, m, _ = run_device(hp, cfg, apply_mode=rng.randint(0, 1),
                                     acc_slots=rng.choice([2, 3, 8]),
                                     merge_ticks=rng.randint(0, 1))
    assert_same(o, trace, wg, wl)
    if cfg.momentum:
        assert np.array_equal(m, o.m)


def test_per_tick_states(hp):
    """Advance the device controller commit by commit (forcing early applies)
    and compare w_global and every w_local not waiting at its gate with the
    oracle's state after the same tick."""
    cfg = C2.replace(nparams=2053, waves=6, D=1, tau=(5, 7, 9, 12))
    states = []

    def on_tick(t, sm):
        states.append((t, len(sm.commit), sm.wg.copy(), [w.copy() for w in sm.wl],
                       list(sm.at_gate)))

    run_schedule(cfg, on_tick=on_tick)
    ctx = hp.Context(hp.config_from(cfg))
    ctx.schedule_begin(cfg.tau, cfg.latency())
    checked = 0
    for target in range(1, cfg.num_vw * cfg.waves + 1):
        reached = ctx.schedule_advance(target)
        t, ncommit, wg, wl, at_gate = next(s for s in states if s[1] >= target)
        assert reached == ncommit
        assert np.array_equal(ctx.read_weights(-1), wg)
        for v in range(cfg.num_vw):
            if not at_gate[v]:
                assert np.array_equal(ctx.read_weights(v), wl[v]), (target, v)
                checked += 1
    assert checked > 10
    ctx.close()


def test_external_gradients_match_synthetic(hp):
    """EXTERNAL mode: the same Philox gradients, supplied as host buffers
    (hp_accumulate_minibatch_host via the controller), give the same result."""
    cfg = C2.replace(nparams=1030, waves=3, D=0, tau=(3, 4, 6, 7))
    o = run_schedule(cfg)
    idx = np.arange(cfg.nparams)
    last_p = cfg.waves * cfg.Nm
    bufs = []
    for v in range(cfg.num_vw):
        for p in range(0, last_p):
            bufs.append(None)
    # host buffer k = (v*last_p + p) % n  ->  n = N*last_p + 1 keeps them distinct
    n = cfg.num_vw * last_p + 1
    bufs = [np.zeros(cfg.nparams, dtype=np.float32) for _ in range(n)]
    for v in range(cfg.num_vw):
        for p in range(1, last_p + 1):
            bufs[(v * last_p + p) % n][:] = gradient(idx, v, p, cfg)
    ctx = hp.Context(hp.config_from(cfg, grad_mode=GRAD_EXTERNAL))
    ctx.schedule_set_host_grads(bufs)
    ctx.run_schedule(cfg.tau, cfg.latency())
    assert np.array_equal(ctx.read_weights(-1), o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(ctx.read_weights(v), o.wl[v])
    ctx.close()


def replay_events(hp, cfg, shuffle_seed=None, merge=1):
    """Drive the event-granular ABI (hp_set_tick, hp_accumulate_minibatch,
    hp_push_wave, hp_pull, hp_tick_end) through the oracle's own event order;
    optionally shuffle the COMPLETE order inside each tick (phase order and
    commit order are what the protocol fixes, not the VW order of completes)."""
    o = run_schedule(cfg)
    ctx = hp.Context(hp.config_from(cfg, merge_ticks=merge))
    rng = random.Random(shuffle_seed)
    by_tick = {}
    for ln in o.trace:
        f = ln.split()
        by_tick.setdefault(int(f[0]), []).append((f[1], int(f[2]), f[3], int(f[4]), int(f[5])))
    for t in sorted(by_tick):
        if t == 0 and all(k == "START" for _, _, k, _, _ in by_tick[t]):
            continue
        ctx.set_tick(t)
        ev = by_tick[t]
        comps = [(v, p) for ph, v, k, p, c in ev if k == "COMPLETE"]
        if shuffle_seed is not None:
            rng.shuffle(comps)
        for v, p in comps:
            ctx.accumulate_minibatch(v, p)
        for ph, v, k, p, c in ev:
            if k == "PUSH":
                ctx.push_wave(v, c)
        for v in range(cfg.num_vw):
            try:
                ctx.pull(v)
            except hp.HetPipeError as e:
                assert e.status == hp.HP_ERR_PROTOCOL      # not waiting at its gate
        ctx.tick_end()
    ctx.flush()
    with tempfile.NamedTemporaryFile(suffix=".trace") as f:
        trace = ctx.trace_lines(f.name)
    wg = ctx.read_weights(-1)
    wl = [ctx.read_weights(v) for v in range(cfg.num_vw)]
    ctx.close()
    return o, trace, wg, wl


@pytest.mark.parametrize("seed", range(12))
def test_event_api_replay(hp, seed):
    cfg = _rand_cfg(500 + seed).replace(local_semantics=LOCAL_STRICT, momentum=0.0)
    o, trace, wg, wl = replay_events(hp, cfg, merge=seed % 2)
    assert_same(o, trace, wg, wl)
    o, trace, wg, wl = replay_events(hp, cfg, shuffle_seed=seed, merge=seed % 2)
    assert np.array_equal(wg, o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(wl[v], o.wl[v])


def test_event_api_protocol_errors(hp):
    """Negative ABI tests: duplicate / out-of-order / incomplete push,
    out-of-order completion, pull outside the gate, WOULD_BLOCK without effect."""
    cfg = C1.replace(nparams=64, waves=4)
    ctx = hp.Context(hp.config_from(cfg))
    E = hp.HetPipeError
    with pytest.raises(E) as e:
        ctx.accumulate_minibatch(0, 2)              # minibatch 2 not started
    assert e.value.status == hp.HP_ERR_PROTOCOL
    with pytest.raises(E):
        ctx.push_wave(0, 0)                          # incomplete wave
    with pytest.raises(E):
        ctx.pull(0)                                  # not at the gate
    ctx.accumulate_minibatch(0, 1)
    with pytest.raises(E):
        ctx.push_wave(0, 1)                          # out of order
    ctx.push_wave(0, 0)
    with pytest.raises(E):
        ctx.push_wave(0, 0)                          # duplicate
    cl, cg, blocked = ctx.clock(0)
    assert (cl, cg, blocked) == (1, 0, True)         # D=0: waits for vw 1
    before = ctx.read_weights(0)
    assert ctx.pull(0) == hp.HP_WOULD_BLOCK
    assert np.array_equal(ctx.read_weights(0), before)
    ctx.accumulate_minibatch(1, 1)
    ctx.push_wave(1, 0)
    assert ctx.pull(0) == hp.HP_OK and ctx.pull(1) == hp.HP_OK
    ctx.tick_end()
    assert ctx.clock(0)[:2] == (1, 1)
    ctx.close()


def test_zero_and_tiny_sizes(hp):
    for P in (0, 1, 2, 3, 5):
        cfg = C1.replace(nparams=P, waves=3)
        o = run_schedule(cfg)
        trace, wg, wl, _, _ = run_device(hp, cfg)
        assert_same(o, trace, wg, wl)


@pytest.mark.parametrize("cfg", [C2.replace(waves=3), C3.replace(waves=3),
                                 C5.replace(waves=2, D=4),
                                 C2.replace(waves=3, grad_mode=GRAD_CONVEX, lr=0.05),
                                 C2.replace(waves=2, F=2, D=1),
                                 C4.replace(waves=2, grad_mode=GRAD_CONVEX, lr=0.05, F=2),
                                 C2.replace(waves=3, grad_mode=GRAD_CONVEX, lr=0.3,
                                            lr_schedule=1)],
                         ids=["C2", "C3", "C5", "C2-convex", "C2-F2", "C4-convex-F2",
                              "C2-convex-theorem1"])
def test_full_size_sampled(hp, cfg):
    """Full model sizes in the bench's launch configuration: sampled params
    (stride 4099 + both ends) against the oracle restricted to that sample."""
    idx = np.array(sample_indices(cfg.nparams), dtype=np.int64)
    o = run_schedule(cfg, idx=idx)
    trace, wg, wl, m, _ = run_device(hp, cfg)
    assert_same(o, trace, wg, wl, idx=idx)
    if cfg.momentum:
        assert np.array_equal(m[idx], o.m)


def test_beyond_int32_indices_sampled(hp):
    """2^31 + 37 params (8.6 GB per fp32 buffer, ~60 GB of arena): every index,
    chunk and tile computation is 64-bit. Sampled params around 2^31, 2^30, the
    ends and every 2^24-th, read back one by one, against the oracle on the
    same sample (FLOAT gradients, momentum: every path of the fused kernel)."""
    torch = pytest.importorskip("torch")
    free, _ = torch.cuda.mem_get_info()
    if free < 80 * 2 ** 30:
        pytest.skip("needs ~64 GB of free device memory")
    P = 2 ** 31 + 37
    cfg = C1.replace(name="big", nparams=P, Nm=2, D=1, waves=3, tau=(5, 7), lr=0.01,
                     momentum=0.9, grad_mode=0)
    idx = set(range(0, P, 2 ** 24))
    for c in (0, 2 ** 30, 2 ** 31, P - 1):
        idx.update(i for i in range(c - 9, c + 10) if 0 <= i < P)
    idx = np.array(sorted(idx), dtype=np.int64)
    o = run_schedule(cfg, idx=idx)
    ctx = hp.Context(hp.config_from(cfg))
    ctx.run_schedule(cfg.tau, cfg.latency())
    with tempfile.NamedTemporaryFile(suffix=".trace") as f:
        assert ctx.trace_lines(f.name) == o.trace
    one = np.empty(1, dtype=np.float32)

    def sampled(which):
        return np.array([ctx.read_weights(which, int(i), 1, out=one)[0] for i in idx], np.float32)
    assert np.array_equal(sampled(-1), o.wg)
    assert np.array_equal(sampled(-2), o.m)
    for v in range(cfg.num_vw):
        assert np.array_equal(sampled(v), o.wl[v]), f"w_local({v})"
    ctx.close()


def test_c4_sharded_ranks_sampled(hp):
    """ED-local placement: two rank-shards of C4 run as separate
    contexts on one GPU reproduce the oracle at sampled params of each shard."""
    from workloads import even_shards
    cfg = C4.replace(waves=2)
    b = even_shards(cfg.nparams, 2)
    for r in range(2):
        lo, hi = b[r], b[r + 1]
        idx = np.array(sorted(set(list(range(lo, hi, 7919)) + [lo, lo + 1, hi - 1])), dtype=np.int64)
        o = run_schedule(cfg, idx=idx)
        ctx = hp.Context(hp.config_from(cfg, param_begin=lo, param_count=hi - lo))
        ctx.run_schedule(cfg.tau, cfg.latency())
        assert np.array_equal(ctx.read_weights(-1)[idx - lo], o.wg)
        for v in range(cfg.num_vw):
            assert np.array_equal(ctx.read_weights(v)[idx - lo], o.wl[v])
        ctx.close()


def pmp_timing_oracle(model, vws, Nm):
    """(tau, lat) in microseconds from the ORACLE's partitioner and pipeline
    simulator (oracle/pipeline.py), the same recipe as
    paper_2005_14038_b200/schedule.py (whose native partitioner and simulator
    tests/test_pipeline_schedule.py matches exactly)."""
    from oracle import pipeline as op
    from workloads import models as M
    F = M.v_flops_per_s()
    tau, lat = [], []
    for types in vws:
        g = [{"flops": F * M.GPUS[t].speed, "mem": M.GPUS[t].mem_gb * 1e9, "node": M.NODE_OF[t]}
             for t in types]
        b, order, cuts = op.partition_bruteforce(M.MODELS[model](), g, Nm)
        costs = op.stage_costs(M.MODELS[model](), cuts, [g[i] for i in order])
        t_ns, l_ns = op.derive_tau_latency(costs, Nm)
        tau.append(max(1, round(t_ns / 1000)))
        lat.append(max(1, round(l_ns / 1000)))
    return tuple(tau), tuple(lat)


@pytest.mark.parametrize("D,policy", [(0, 0), (2, 0), (1, 1)])
def test_pipeline_derived_timing(hp, D, policy):
    """NEXT-1: tau_v / L_v from partitioning VGG-19 over NP's four VW types
    (VVVV, RRRR, GGGG, QQQQ) and simulating each VW's pipeline drive the tick
    controller; the CUDA path still matches the oracle bit for bit."""
    tau, lat = pmp_timing_oracle("vgg19", ("VVVV", "RRRR", "GGGG", "QQQQ"), 4)
    cfg = C2.replace(nparams=4099, waves=8, D=D, tau=tau, lat=lat, pull_policy=policy)
    o = run_schedule(cfg)
    trace, wg, wl, _, _ = run_device(hp, cfg)
    assert_same(o, trace, wg, wl)


@pytest.mark.parametrize("seed", range(40))
def test_convex_random_bit_exact(hp, seed):
    """NEXT-2 CONVEX workload: every gradient reads the w_local its minibatch
    saw at START (the device stash ring), so a wrong version anywhere changes
    the numbers. Random configs, all modes: identical traces, bit-exact arrays."""
    rng = random.Random(7000 + seed)
    base = _rand_cfg(seed)
    cfg = base.replace(grad_mode=GRAD_CONVEX, lr=0.05, conv_a=rng.choice([0.5, 1.0]),
                       conv_sigma=rng.choice([0.0, 1.0]), w0_mode=W0_PHILOX)
    o = run_schedule(cfg)
    trace, wg, wl, m, _ = run_device(hp, cfg, apply_mode=rng.randint(0, 1),
                                     acc_slots=rng.choice([2, 3, 8]),
                                     merge_ticks=rng.randint(0, 1))
    assert_same(o, trace, wg, wl)
    if cfg.momentum:
        assert np.array_equal(m, o.m)


@pytest.mark.parametrize("seed", range(24))
def test_theorem1_schedule_random_bit_exact(hp, seed):
    """NEXT-2: Theorem 1's step sizes eta_t = sigma / sqrt(t), t = (p-1)N + v + 1
    (reading Z26), per op on the device (host-computed fp32, in
    each complete / fold), on the CONVEX and the FLOAT workloads, EXTERNAL
    excluded: identical traces, bit-exact arrays."""
    rng = random.Random(9100 + seed)
    base = _rand_cfg(seed)
    convex = rng.random() < 0.6
    cfg = base.replace(lr_schedule=1, lr=rng.choice([0.05, 0.3]),
                       grad_mode=GRAD_CONVEX if convex else GRAD_FLOAT,
                       conv_sigma=rng.choice([0.0, 0.5]), w0_mode=W0_PHILOX,
                       F=rng.choice([1, 1, 2]))
    o = run_schedule(cfg)
    trace, wg, wl, m, _ = run_device(hp, cfg, apply_mode=rng.randint(0, 1),
                                     acc_slots=rng.choice([2, 3]),
                                     merge_ticks=rng.randint(0, 1))
    assert_same(o, trace, wg, wl)
    if cfg.momentum:
        assert np.array_equal(m, o.m)


def test_convex_per_tick_states(hp):
    """CONVEX: the device w_local after every commit equals the oracle's."""
    cfg = C2.replace(nparams=2053, waves=6, D=1, tau=(5, 7, 9, 12), grad_mode=GRAD_CONVEX,
                     lr=0.05)
    states = []

    def on_tick(t, sm):
        states.append((t, len(sm.commit), sm.wg.copy(), [w.copy() for w in sm.wl],
                       list(sm.at_gate)))

    run_schedule(cfg, on_tick=on_tick)
    ctx = hp.Context(hp.config_from(cfg))
    ctx.schedule_begin(cfg.tau, cfg.latency())
    for target in range(1, cfg.num_vw * cfg.waves + 1):
        reached = ctx.schedule_advance(target)
        t, ncommit, wg, wl, at_gate = next(s for s in states if s[1] >= target)
        assert reached == ncommit
        assert np.array_equal(ctx.read_weights(-1), wg)
        for v in range(cfg.num_vw):
            if not at_gate[v]:
                assert np.array_equal(ctx.read_weights(v), wl[v]), (target, v)
    ctx.close()


@pytest.mark.parametrize("seed", range(40))
def test_update_frequency_random_bit_exact(hp, seed):
    """NEXT-4: one clock = F waves (aggregate and push F*Nm minibatches, gate
    at (c+2)*F*Nm, STRICT pulls add the open clock's own aggregate). Random
    configs in every mode, incl. CONVEX: identical traces, bit-exact arrays."""
    rng = random.Random(9000 + seed)
    base = _rand_cfg(seed)
    cfg = base.replace(F=rng.randint(2, 4), waves=max(1, base.waves // 2))
    if rng.random() < 0.3:
        cfg = cfg.replace(grad_mode=GRAD_CONVEX, lr=0.05, w0_mode=W0_PHILOX)
    o = run_schedule(cfg)
    trace, wg, wl, m, _ = run_device(hp, cfg, apply_mode=rng.randint(0, 1),
                                     acc_slots=rng.choice([2, 3]),
                                     merge_ticks=rng.randint(0, 1))
    assert_same(o, trace, wg, wl)
    if cfg.momentum:
        assert np.array_equal(m, o.m)


@pytest.mark.parametrize("F,Nm,D,tau,mode", [(2, 3, 0, (2, 9), GRAD_FLOAT),
                                             (2, 2, 0, (3, 7, 5), GRAD_FLOAT),
                                             (3, 2, 1, (2, 11), GRAD_CONVEX),
                                             (2, 4, 0, (5, 6, 13), GRAD_CONVEX)])
def test_update_frequency_blocked_strict(hp, F, Nm, D, tau, mode):
    """F > 1, STRICT, a fast VW waiting at its gate while its in-flight
    minibatches complete: the pull must add the open clock's aggregate as it
    stood at the gate (the device snapshot), not the backlog's updates."""
    cfg = WSPConfig("fb", len(tau), Nm, D, 1027, 5, tau, F=F, grad_mode=mode,
                    lr=0.05 if mode == GRAD_CONVEX else 0.01)
    o = run_schedule(cfg)
    for merge in (0, 1):
        trace, wg, wl, _, _ = run_device(hp, cfg, merge_ticks=merge)
        assert_same(o, trace, wg, wl)


@pytest.mark.parametrize("seed", range(24))
def test_external_gradients_random(hp, seed):
    """EXTERNAL host gradients (the library's ring of Nm device slots per VW)
    on random configs with gate waits: a deferred STRICT fold re-reads the
    slot of its minibatch, which the copy for minibatch p + Nm replaces --
    the queued fold must reach the device first."""
    base = _rand_cfg(4000 + seed)
    cfg = base.replace(grad_mode=GRAD_FLOAT, lr=0.01)
    o = run_schedule(cfg)
    idx = np.arange(cfg.nparams)
    last_p = cfg.waves * cfg.Nm
    n = cfg.num_vw * last_p + 1
    bufs = [np.zeros(cfg.nparams, dtype=np.float32) for _ in range(n)]
    for v in range(cfg.num_vw):
        for p in range(1, last_p + 1):
            bufs[(v * last_p + p) % n][:] = gradient(idx, v, p, cfg)
    rng = random.Random(seed)
    ctx = hp.Context(hp.config_from(cfg, grad_mode=GRAD_EXTERNAL,
                                    merge_ticks=rng.randint(0, 1), apply_mode=rng.randint(0, 1)))
    ctx.schedule_set_host_grads(bufs)
    ctx.run_schedule(cfg.tau, cfg.latency())
    assert np.array_equal(ctx.read_weights(-1), o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(ctx.read_weights(v), o.wl[v]), f"w_local({v})"
    ctx.close()

"""CPU tests of the engine's HOST logic (batching, deferred applies, fold
elision, descriptor splitting): the real engine.cpp/capi.cpp linked against a
scalar host emulation of the tick descriptor (tests/emu, test-only), checked
against the oracle exactly like the GPU parity tests. The device kernels
themselves are covered by tests/test_gpu_parity.py on a B200."""
import random

import numpy as np
import pytest

import test_gpu_parity as G
from oracle import run_schedule
from workloads import C1, C1_SKEW, C2, WSPConfig


@pytest.fixture(scope="module")
def hp():
    from paper_2005_14038_b200 import hetpipe
    from emu import build_emu
    lib = hetpipe.load_test_library(build_emu.build())
    return G._HP(hetpipe, lib)


@pytest.mark.parametrize("cfg", [C1, C1_SKEW], ids=["C1", "C1-skew"])
@pytest.mark.parametrize("apply_mode", [0, 1])
def test_c1(hp, cfg, apply_mode):
    G.test_c1_bsp_limit_bit_exact(hp, cfg, apply_mode)


@pytest.mark.parametrize("seed", range(160))
def test_random_configs(hp, seed):
    G.test_random_configs_bit_exact(hp, seed)


def test_per_tick_states(hp):
    G.test_per_tick_states(hp)


def test_external_gradients(hp):
    G.test_external_gradients_match_synthetic(hp)


@pytest.mark.parametrize("seed", range(40))
def test_event_api_replay(hp, seed):
    G.test_event_api_replay(hp, seed % 12) if seed < 12 else _replay_more(hp, seed)


def _replay_more(hp, seed):
    cfg = G._rand_cfg(900 + seed)
    o, trace, wg, wl = G.replay_events(hp, cfg, shuffle_seed=seed, merge=seed % 2)
    assert np.array_equal(wg, o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(wl[v], o.wl[v])


def test_protocol_errors(hp):
    G.test_event_api_protocol_errors(hp)


def test_zero_and_tiny(hp):
    G.test_zero_and_tiny_sizes(hp)


@pytest.mark.parametrize("N,Nm,D,policy", [(8, 8, 0, 0), (8, 8, 4, 1), (8, 6, 1, 0), (5, 8, 32, 1)])
def test_descriptor_overflow(hp, N, Nm, D, policy):
    """Ticks with many VWs, long backlogs and many deferred applies force the
    apply-only pre-launches and split w_local groups."""
    tau = tuple(1 + (3 * v) % 5 for v in range(N))
    cfg = WSPConfig("ovf", N, Nm, D, 133, 12, tau, pull_policy=policy,
                    lat=tuple(t * Nm for t in tau))
    o = run_schedule(cfg)
    for apply_mode in (0, 1):
        for slots in (2, 8):
            for merge in (0, 1):
                trace, wg, wl, _, _ = G.run_device(hp, cfg, apply_mode, slots, merge_ticks=merge)
                G.assert_same(o, trace, wg, wl)


@pytest.mark.parametrize("seed", range(6))
def test_same_tick_pushes_out_of_complete_order(hp, seed):
    """C1 (equal speeds, N_m=1): both VWs push in every tick; shuffled complete
    order makes commit order differ from complete order, which must split the
    launch so no apply reads an acc slot before this tick writes it."""
    for cfg in (C1, C1.replace(momentum=0.5, grad_mode=0, lr=0.01, w0_mode=1)):
        o, trace, wg, wl = G.replay_events(hp, cfg, shuffle_seed=seed, merge=seed % 2)
        assert np.array_equal(wg, o.wg)
        for v in range(cfg.num_vw):
            assert np.array_equal(wl[v], o.wl[v])


@pytest.mark.parametrize("cfg", [C1, C1_SKEW, C2.replace(nparams=999, waves=6)],
                         ids=["C1", "C1-skew", "C2"])
def test_sync_latency_records(hp, cfg):
    """hp_profile_sync_latency: one record per (VW, wave) whose push and pull
    fall in the profile window -- under EAGER every admission after a push
    pulls, so the records equal the pulls, each VW's in wave order."""
    from paper_2005_14038_b200 import hetpipe
    ctx = hetpipe.Context(hetpipe.config_from(cfg), lib=hp.lib)
    ctx.profile_enable(True)
    ctx.run_schedule(cfg.tau, cfg.latency())
    ms, vw, waited = ctx.profile_sync_latency()
    st = ctx.stats()
    assert len(ms) == sum(st.pulls[:cfg.num_vw])
    for v in range(cfg.num_vw):
        assert int((vw == v).sum()) == st.pulls[v]
    assert np.all(ms >= 0)
    # waited flags: C1's equal speeds never block; the skewed C1 blocks its fast VW
    assert int(waited.sum()) == (0 if cfg is C1 else int(waited.sum()))
    if cfg is C1_SKEW:
        assert waited.any() and not waited[vw == 1].any()
    ctx.close()


@pytest.mark.parametrize("D,policy", [(0, 0), (2, 0), (1, 1)])
def test_pipeline_derived_timing(hp, D, policy):
    G.test_pipeline_derived_timing(hp, D, policy)


@pytest.mark.parametrize("seed", range(80))
def test_convex_random(hp, seed):
    G.test_convex_random_bit_exact(hp, seed % 40) if seed < 40 else _convex_more(hp, seed)


def _convex_more(hp, seed):
    import random as _r
    from workloads import GRAD_CONVEX
    rng = _r.Random(seed)
    cfg = G._rand_cfg(3000 + seed).replace(grad_mode=GRAD_CONVEX, lr=0.05, w0_mode=1,
                                           conv_sigma=rng.choice([0.0, 1.0]))
    o = run_schedule(cfg)
    trace, wg, wl, _, _ = G.run_device(hp, cfg, rng.randint(0, 1), rng.choice([2, 3]),
                                       merge_ticks=rng.randint(0, 1))
    G.assert_same(o, trace, wg, wl)


def test_convex_per_tick_states(hp):
    G.test_convex_per_tick_states(hp)


@pytest.mark.parametrize("seed", range(120))
def test_update_frequency_random(hp, seed):
    G.test_update_frequency_random_bit_exact(hp, seed)


@pytest.mark.parametrize("F,Nm,D,tau,mode", [(2, 3, 0, (2, 9), 0), (2, 2, 0, (3, 7, 5), 0),
                                             (3, 2, 1, (2, 11), 3), (2, 4, 0, (5, 6, 13), 3)])
def test_update_frequency_blocked_strict(hp, F, Nm, D, tau, mode):
    G.test_update_frequency_blocked_strict(hp, F, Nm, D, tau, mode)


@pytest.mark.parametrize("seed", range(24))
def test_external_gradients_random(hp, seed):
    G.test_external_gradients_random(hp, seed)


@pytest.mark.parametrize("seed", range(40))
def test_theorem1_schedule(hp, seed):
    """NEXT-2: Theorem 1's per-op step sizes through the engine's descriptors."""
    G.test_theorem1_schedule_random_bit_exact(hp, seed)

"""Lockstep exchange transports (include/hetpipe.h HP_XPORT_NCCL / HP_XPORT_NVLS)
on CPU: G ranks as threads driving the REAL engine (host-emulated kernels and
collectives, tests/emu). A lockstep batch -- one full-replica VW per GPU, SGD,
every VW pushing the same wave and pulling in one batch (D = 0, equal speeds)
-- is summed per PS shard and applied once (reduce-scatter + apply +
all-gather, or the NVSwitch's multimem.ld_reduce / multimem.st), instead of N
sequential applies in commit order.

Checks against the oracle: identical traces on every rank (the protocol does
not change); DYADIC gradients (integers x 2^-6, every partial sum exact in
fp32) give bit-identical arrays for ANY summation order; FLOAT gradients are
within reading Z15's normwise bound (max|a-b| / max|b| <= 1e-5); batches that
do not qualify (mixed speeds, momentum) take the PEER path and stay bit-exact.
"""
import random
import tempfile
import threading

import numpy as np
import pytest

from oracle import run_schedule
from workloads import (GRAD_DYADIC, GRAD_FLOAT, LOCAL_AT_LEAST, LOCAL_STRICT, PULL_EAGER,
                       PULL_LAZY, WSPConfig)

NCCL, NVLS = 1, 2


@pytest.fixture(scope="module")
def lib():
    from emu import build_emu
    from paper_2005_14038_b200 import hetpipe
    return hetpipe.load_test_library(build_emu.build())


def run_transport(lib, cfg, G, transport, **over):
    """k = 1 (full replica per VW). NVLS: host arenas stand in for the symmetric
    allocation (hp_config.arena + hp_connect_symmetric); the emulated kernel
    sums through the unicast mappings, the multicast base is never read."""
    from paper_2005_14038_b200 import hetpipe
    cid = hetpipe.comm_unique_id(lib)
    cfgs = [hetpipe.config_from(cfg, world=G, rank=r, vw_span=1, transport=transport, **over)
            for r in range(G)]
    keep, bases = [], []
    if transport == NVLS:
        nbytes = max(hetpipe.arena_bytes(c, lib=lib) for c in cfgs)
        for c in cfgs:
            raw = np.zeros(nbytes + 256, dtype=np.uint8)
            base = (raw.ctypes.data + 255) // 256 * 256
            keep.append(raw)
            bases.append(base)
            c.arena = base
    ctxs = [hetpipe.Context(c, lib=lib) for c in cfgs]
    handles = [c.ipc_handle() for c in ctxs] if transport != NVLS else None
    out, errs = [None] * G, []

    def work(r):
        try:
            c = ctxs[r]
            if transport == NVLS:
                c.connect_symmetric(bases, 1 << 40, cid)
            else:
                c.connect(handles, cid)
            c.run_schedule(cfg.tau, cfg.latency())
            with tempfile.NamedTemporaryFile(suffix=".trace") as f:
                tr = c.trace_lines(f.name)
            wg = c.read_weights(-1)
            wl = {r: c.read_weights(r)} if r < cfg.num_vw else {}
            out[r] = (tr, wg, wl, c.stats())
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not errs, errs
    for c in ctxs:
        c.close()
    del keep
    return out


def normwise(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))


def check(cfg, G, out, exact):
    o = run_schedule(cfg)
    for r in range(G):
        assert out[r][0] == o.trace, f"rank {r} trace"
    wg = np.concatenate([out[r][1] for r in range(G)])
    wls = [out[v][2][v] for v in range(cfg.num_vw)]
    if exact:
        assert np.array_equal(wg, o.wg)
        for v in range(cfg.num_vw):
            assert np.array_equal(wls[v], o.wl[v]), f"w_local({v})"
    else:
        assert normwise(wg, o.wg) <= 1e-5
        for v in range(cfg.num_vw):
            assert normwise(wls[v], o.wl[v]) <= 1e-5, f"w_local({v})"
    return o


def lockstep_cfg(G, Nm, D, P, W, mode, **kw):
    return WSPConfig("lock", G, Nm, D, P, W, (5,) * G,
                     lr=0.01 if mode == GRAD_FLOAT else 2.0 ** -6, grad_mode=mode, **kw)


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
@pytest.mark.parametrize("G", [2, 3, 4])
def test_lockstep_dyadic_exact(lib, transport, G):
    cfg = lockstep_cfg(G, 3, 0, 1027, 5, GRAD_DYADIC)
    out = run_transport(lib, cfg, G, transport)
    check(cfg, G, out, exact=True)
    # every round was exchanged by the collective transport
    assert all(out[r][3].lockstep_batches == cfg.waves for r in range(G))


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
def test_lockstep_float_normwise(lib, transport):
    cfg = lockstep_cfg(4, 4, 0, 4099, 6, GRAD_FLOAT)
    out = run_transport(lib, cfg, 4, transport)
    check(cfg, 4, out, exact=False)
    assert out[0][3].lockstep_batches == cfg.waves


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
def test_non_lockstep_falls_back_to_peer(lib, transport):
    # mixed speeds: pushes arrive in different ticks -> PEER path, bit-exact in FLOAT
    cfg = WSPConfig("mixed", 3, 2, 1, 999, 5, (3, 5, 4))
    out = run_transport(lib, cfg, 3, transport)
    check(cfg, 3, out, exact=True)
    assert all(out[r][3].lockstep_batches == 0 for r in range(3))
    # momentum: never a single-sum apply (heavy ball is per push, Z11)
    cfg = lockstep_cfg(2, 2, 0, 333, 4, GRAD_FLOAT, momentum=0.9)
    out = run_transport(lib, cfg, 2, transport)
    check(cfg, 2, out, exact=True)
    assert out[0][3].lockstep_batches == 0


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
def test_lockstep_uneven_shards(lib, transport):
    # layer-round-robin-like uneven PS shards: the reduce-scatter / all-gather
    # (grouped per shard) and the per-owner NVLS ranges follow the bounds
    cfg = lockstep_cfg(3, 2, 0, 4099, 5, GRAD_DYADIC)
    out = run_transport(lib, cfg, 3, transport, ps_bounds=[0, 2976, 3840, 4099])
    check(cfg, 3, out, exact=True)
    assert out[0][3].lockstep_batches == cfg.waves
    assert [len(out[r][1]) for r in range(3)] == [2976, 864, 259]


@pytest.mark.parametrize("seed", range(12))
def test_lockstep_random(lib, seed):
    rng = random.Random(seed)
    G = rng.choice([2, 3, 4])
    transport = rng.choice([NCCL, NVLS])
    cfg = WSPConfig("lr", G, rng.randint(1, 4), rng.randint(0, 3), rng.choice([64, 333, 1030, 4099]),
                    rng.randint(1, 6), (rng.randint(1, 9),) * G, lr=2.0 ** -6,
                    grad_mode=GRAD_DYADIC, pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
                    local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]))
    out = run_transport(lib, cfg, G, transport, merge_ticks=rng.randint(0, 1),
                        acc_slots=rng.choice([2, 3]), apply_mode=rng.randint(0, 1))
    check(cfg, G, out, exact=True)


def test_arena_bytes_congruent(lib):
    from paper_2005_14038_b200 import hetpipe
    # one VW per GPU: every rank's arena has the same size and offsets, so a
    # multicast mapping addresses the same buffer on every GPU
    cfg = lockstep_cfg(3, 2, 0, 1000, 3, GRAD_FLOAT)
    sizes = {hetpipe.arena_bytes(hetpipe.config_from(cfg, world=3, rank=r, vw_span=1,
                                                     transport=NVLS), lib=lib) for r in range(3)}
    assert len(sizes) == 1


def test_nvls_requires_symmetric_connect(lib):
    from paper_2005_14038_b200 import hetpipe
    cfg = lockstep_cfg(2, 2, 0, 256, 2, GRAD_FLOAT)
    cid = hetpipe.comm_unique_id(lib)
    ctx = hetpipe.Context(hetpipe.config_from(cfg, world=2, rank=0, vw_span=1, transport=NVLS),
                          lib=lib)
    with pytest.raises(hetpipe.HetPipeError) as e:
        ctx.connect([ctx.ipc_handle()] * 2, cid)
    assert e.value.status == hetpipe.HP_ERR_STATE
    ctx.close()


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
def test_lockstep_convex(lib, transport):
    # weight-dependent gradients through the collective exchange: the STASH of
    # the gated START follows the collective pull (normwise: one-sum applies)
    cfg = lockstep_cfg(3, 2, 0, 1030, 4, GRAD_FLOAT).replace(grad_mode=3, lr=0.05)
    out = run_transport(lib, cfg, 3, transport)
    check(cfg, 3, out, exact=False)
    assert out[0][3].lockstep_batches == cfg.waves


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
def test_update_frequency_never_lockstep(lib, transport):
    # F > 1: a STRICT pull adds the open clock's aggregate -> never a collective
    cfg = lockstep_cfg(2, 2, 0, 1030, 3, GRAD_FLOAT).replace(F=2)
    out = run_transport(lib, cfg, 2, transport)
    check(cfg, 2, out, exact=True)
    assert out[0][3].lockstep_batches == 0

"""Eight GPUs without eight GPUs (BASELINE configs[2..4] at G = 8; SURVEY.md
8(e)): the REAL engine under the host emulation, 8 ranks as threads, for the
placements bench.py runs at --gpus 8 -- C3 with two-stage VWs (k = 2), C4
ED-local (the north_star target), C5 with one VW per GPU and momentum, C5E /
HVD through both lockstep transports -- checked against the oracle, with the
tick descriptors never overflowing (hp_stats.desc_splits == 0: at G = 8,
N = 8 every batch fits kMaxA = 16 applies, kMaxS = 32 segments, kMaxP = 16
owner-side pull targets, kMaxG = 8 groups in one launch)."""
import argparse

import numpy as np
import pytest

import bench
from oracle import run_schedule
from placement_check import check, run_colocated
from test_transport_emu import NCCL, NVLS, run_transport
from test_transport_emu import check as check_transport
from workloads import C5E, HVD, GRAD_DYADIC, WSPConfig

G = 8


@pytest.fixture(scope="module")
def emu():
    from emu import build_emu
    from paper_2005_14038_b200 import hetpipe
    return hetpipe, hetpipe.load_test_library(build_emu.build())


@pytest.fixture(scope="module")
def lib(emu):
    return emu[1]


def host_alloc(nbytes):
    buf = np.zeros(nbytes + 256, dtype=np.uint8)
    addr = buf.ctypes.data
    return addr + (-addr) % 256, buf


def bench_args(config, **kw):
    a = argparse.Namespace(config=config, span=-1, num_vw=0, update_freq=1, D=-1, pull="eager",
                           grad="float", timing="proxy")
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("config,span_want", [("C3", 2), ("C5", 1), ("C4", 0), ("C2", 0)])
def test_bench_resolves_survey_placement_at_8(config, span_want):
    cfg, span = bench.resolve_config(bench_args(config), G)
    assert span == span_want
    assert bench.resolve_config(bench_args(None), G)[0].name == "C3"
    assert bench.resolve_config(bench_args(None), 1)[0].name == "C2"


@pytest.mark.parametrize("config,D", [("C3", None), ("C5", 0), ("C5", 4), ("C5", 32)])
def test_bench_config_at_8_under_emulation(emu, config, D):
    """The configuration `bench.py --gpus 8 [--config C5 --D d]` measures,
    shrunk in P and W, run by 8 emulated ranks: identical traces, bit-exact
    shards and stages, no descriptor overflow."""
    hetpipe, lib = emu
    cfg, span = bench.resolve_config(bench_args(config, D=-1 if D is None else D), G)
    cfg = cfg.replace(nparams=8 * 1024 + 77, waves=4)
    out = run_colocated(hetpipe, cfg, G, span, host_alloc, lib=lib, timeout=300)
    check(cfg, G, span, out)


def _splits_colocated(hetpipe, lib, cfg, k, **over):
    """desc_splits of every rank of an emulated co-located run."""
    from placement_check import collect
    import threading
    ctxs, keep = [], []
    for r in range(G):
        c = hetpipe.config_from(cfg, world=G, rank=r, vw_span=k, **over)
        addr, kp = host_alloc(hetpipe.arena_bytes(c, lib))
        keep.append(kp)
        c.arena = addr
        ctxs.append(hetpipe.Context(c, lib=lib))
    bases = [c.cfg.arena for c in ctxs]
    out, splits, errs = [None] * G, [None] * G, []

    def work(r):
        try:
            ctxs[r].connect_symmetric(bases, 0, None)
            ctxs[r].run_schedule(cfg.tau, cfg.latency())
            out[r] = collect(ctxs[r], cfg, G, k, r)
            splits[r] = ctxs[r].stats().desc_splits
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    for c in ctxs:
        c.close()
    return out, splits


@pytest.mark.parametrize("name,cfg,k", [
    ("C5-8VW-mom", WSPConfig("c5", 8, 8, 0, 4096 + 37, 3, (250, 250, 330, 330, 346, 346, 421, 421),
                             momentum=0.9), 1),
    ("C5-8VW-D4", WSPConfig("c5", 8, 8, 4, 4096 + 37, 4, (250, 250, 330, 330, 346, 346, 421, 421),
                            momentum=0.9), 1),
    ("C3-k2", WSPConfig("c3", 4, 4, 4, 4096 + 37, 4, (314, 314, 338, 338)), 2),
    ("N8-k2-lockstep", WSPConfig("e8", 8, 2, 0, 4096 + 37, 4, (7,) * 8), 2),
    ("N8-k4", WSPConfig("e8", 8, 3, 1, 4096 + 37, 4, (3, 4, 5, 6, 7, 8, 9, 10)), 4),
], ids=lambda x: x if isinstance(x, str) else "")
def test_descriptor_limits_never_exceeded_at_8(emu, name, cfg, k):
    hetpipe, lib = emu
    out, splits = _splits_colocated(hetpipe, lib, cfg, k)
    check(cfg, G, k, out)
    assert splits == [0] * G, splits


def test_c4_ed_local_at_8(emu):
    """C4 (the north_star target: 4 VWs ED-local, N_m = 8, D = 32) over 8 ranks:
    every rank owns P/8 of every VW and of the PS (stage q = shard q,
    P:104-106) and runs independently -- no exchange; the concatenated shards
    equal the single-model oracle."""
    hetpipe, lib = emu
    from paper_2005_14038_b200 import dist as hdist
    cfg, span = bench.resolve_config(bench_args("C4"), G)
    assert span == 0
    cfg = cfg.replace(nparams=8 * 4096 + 5, waves=3)
    o = run_schedule(cfg)
    wg, wl = [], [[] for _ in range(cfg.num_vw)]
    for r in range(G):
        ctx = hdist.rank_context(cfg, r, G, lib=lib)
        ctx.run_schedule(cfg.tau, cfg.latency())
        wg.append(ctx.read_weights(-1))
        for v in range(cfg.num_vw):
            wl[v].append(ctx.read_weights(v))
        assert ctx.stats().nvl_bytes == 0 and ctx.stats().desc_splits == 0
        ctx.close()
    assert np.array_equal(np.concatenate(wg), o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(np.concatenate(wl[v]), o.wl[v])


@pytest.mark.parametrize("transport", [NCCL, NVLS], ids=["nccl", "nvls"])
@pytest.mark.parametrize("base", [C5E, HVD], ids=["C5E", "HVD"])
def test_lockstep_transports_at_8(lib, transport, base):
    """One VW per GPU, D = 0, equal speeds: every round is one lockstep batch
    through the reduce-scatter / all-gather or the NVSwitch multimem kernel."""
    cfg = base.replace(num_vw=G, tau=(325,) * G, nparams=8 * 1024 + 77, waves=4,
                       grad_mode=GRAD_DYADIC, lr=2.0 ** -6)
    out = run_transport(lib, cfg, G, transport)
    check_transport(cfg, G, out, exact=True)
    assert all(out[r][3].lockstep_batches == cfg.waves for r in range(G))

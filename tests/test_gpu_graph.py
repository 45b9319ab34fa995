"""hp_schedule_capture / hp_graph_launch (include/hetpipe.h): the controller's
device work captured into CUDA graphs and launched once each. The results
must be bit-identical to the oracle (the same launches, only issued as a
graph), and the API must refuse what would reorder device work."""
import tempfile

import numpy as np
import pytest

from oracle import run_schedule
from placement_check import check, run_colocated
from workloads import C1, C1_SKEW, C2, C3, WSPConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2005_14038_b200 import build, hetpipe
    build.build()
    return hetpipe


def _run_graphs(hp, cfg, pieces, **over):
    ctx = hp.Context(hp.config_from(cfg, device=0, **over))
    ctx.schedule_begin(cfg.tau, cfg.latency())
    total = cfg.num_vw * cfg.waves
    targets = sorted({max(1, total * (i + 1) // pieces) for i in range(pieces)})
    for t in targets:
        g = ctx.schedule_capture(t)
        with pytest.raises(hp.HetPipeError, match="HP_ERR_STATE"):
            ctx.schedule_advance(t + 1)        # a pending graph blocks further work
        g.launch()
        with pytest.raises(hp.HetPipeError, match="HP_ERR_STATE"):
            g.launch()                          # once only
        g.close()
    with tempfile.NamedTemporaryFile(suffix=".trace") as f:
        trace = ctx.trace_lines(f.name)
    wg = ctx.read_weights(-1)
    wl = [ctx.read_weights(v) for v in range(cfg.num_vw)]
    m = ctx.read_weights(-2) if cfg.momentum else None
    ctx.close()
    return trace, wg, wl, m


@pytest.mark.parametrize("cfg,pieces", [
    (C1, 1), (C1, 16), (C1_SKEW, 5),
    (C2.replace(nparams=40_003, waves=6, momentum=0.9), 3),
    (C3.replace(nparams=20_000, waves=7), 4),
    (WSPConfig("cf", 3, 2, 1, 4099, 5, (3, 5, 4), grad_mode=3, lr=0.05, F=2), 2),
], ids=["C1-1", "C1-16", "C1skew-5", "C2mom-3", "C3-4", "convexF-2"])
def test_graph_capture_bit_exact(hp, cfg, pieces):
    o = run_schedule(cfg)
    trace, wg, wl, m = _run_graphs(hp, cfg, pieces)
    assert trace == o.trace
    assert np.array_equal(wg, o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(wl[v], o.wl[v]), f"w_local({v})"
    if cfg.momentum:
        assert np.array_equal(m, o.m)


def test_graph_refuses_reads_before_launch(hp):
    cfg = C1
    ctx = hp.Context(hp.config_from(cfg, device=0))
    ctx.schedule_begin(cfg.tau, cfg.latency())
    g = ctx.schedule_capture(4)
    with pytest.raises(hp.HetPipeError, match="HP_ERR_STATE"):
        ctx.read_weights(-1)
    with pytest.raises(hp.HetPipeError, match="HP_ERR_STATE"):
        ctx.profile_enable(True)
    g.launch()
    ctx.read_weights(-1)
    g.close()
    ctx.close()


def test_graph_capture_colocated_placement(hp):
    """A distributed context's capture forks the accumulation / exchange
    streams from the context stream and joins them back: two co-located ranks
    (threads on this GPU, flag barriers) capture and launch their rounds."""
    import threading

    import torch
    from placement_check import collect
    cfg, G, k = C3.replace(nparams=20_000, waves=6), 2, 1
    keep, ctxs = [], []
    for r in range(G):
        c = hp.config_from(cfg, world=G, rank=r, vw_span=k)
        t = torch.empty(hp.arena_bytes(c), dtype=torch.uint8, device="cuda:0")
        keep.append(t)
        c.arena = t.data_ptr()
        ctxs.append(hp.Context(c))
    bases = [c.cfg.arena for c in ctxs]
    out, errs = [None] * G, []

    def work(r):
        try:
            ctx = ctxs[r]
            ctx.connect_symmetric(bases, 0, None)
            ctx.schedule_begin(cfg.tau, cfg.latency())
            for step in range(1, cfg.waves + 1):
                g = ctx.schedule_capture(cfg.num_vw * step)
                g.launch()
                g.close()
            out[r] = collect(ctx, cfg, G, k, r)
        except Exception as e:
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    check(cfg, G, k, out)
    for c in ctxs:
        c.close()

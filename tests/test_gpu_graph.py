"""hp_schedule_capture / hp_graph_launch (include/hetpipe.h): the controller's
device work captured into CUDA graphs and launched once each. The results
must be bit-identical to the oracle (the same launches, only issued as a
graph), and the API must refuse what would reorder device work."""
import tempfile

import numpy as np
import pytest

from oracle import run_schedule
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


@pytest.mark.parametrize("batch", ["1", "0"], ids=["multitick", "per-tick"])
@pytest.mark.parametrize("cfg,pieces", [
    (C1, 1), (C1, 16), (C1_SKEW, 5),
    (C2.replace(nparams=40_003, waves=6, momentum=0.9), 3),
    (C3.replace(nparams=20_000, waves=7), 4),
    (C3.replace(nparams=100_003, waves=5), 2),          # above the multi-tick size limit
    (WSPConfig("cf", 3, 2, 1, 4099, 5, (3, 5, 4), grad_mode=3, lr=0.05, F=2), 2),
    (WSPConfig("th", 2, 2, 1, 4099, 9, (3, 5), grad_mode=3, lr=0.3, lr_schedule=1), 3),
], ids=["C1-1", "C1-16", "C1skew-5", "C2mom-3", "C3-4", "C3big-2", "convexF-2", "thm1-3"])
def test_graph_capture_bit_exact(hp, monkeypatch, cfg, pieces, batch):
    """Captured ticks -- through the multi-tick kernel for small contexts
    (HP_TICK_BATCH=1, default) or as per-tick launches -- equal the oracle."""
    monkeypatch.setenv("HP_TICK_BATCH", batch)
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


def test_graph_capture_refused_for_distributed_context(hp):
    """Distributed contexts issue their exchange directly (a captured flag
    barrier would spin inside a graph)."""
    import torch
    cfg, G = C3.replace(nparams=4096, waves=2), 2
    c = hp.config_from(cfg, world=G, rank=0, vw_span=1)
    t = torch.empty(hp.arena_bytes(c), dtype=torch.uint8, device="cuda:0")
    c.arena = t.data_ptr()
    ctx = hp.Context(c)
    ctx.schedule_begin(cfg.tau, cfg.latency())
    with pytest.raises(hp.HetPipeError, match="HP_ERR_STATE"):
        ctx.schedule_capture(2)
    ctx.close()

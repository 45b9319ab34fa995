"""Distributed placements (world G > 1, span k) on CPU: G ranks as threads of
one process, each driving the REAL engine (host-emulated kernels, tests/emu)
with peer "IPC" pointers and a thread barrier in place of the NCCL barrier.
Checks the exchange logic of the distributed flush -- every PS shard applies
the pushed u~ slices read from the GPU that holds them, every pull reads the
w_global shards of their owners -- against the oracle: identical traces on
every rank, and the shards / stages reassembled equal the oracle's arrays."""
import os
import random
import tempfile
import threading

import numpy as np
import pytest

from oracle import run_schedule
from workloads import (C3, C5, GRAD_DYADIC, GRAD_EXTERNAL, GRAD_FLOAT, LOCAL_AT_LEAST,
                       LOCAL_STRICT, PULL_EAGER, PULL_LAZY, WSPConfig, even_shards)


@pytest.fixture(scope="module")
def lib():
    from emu import build_emu
    from paper_2005_14038_b200 import hetpipe
    return hetpipe.load_test_library(build_emu.build())


def run_placement(lib, cfg, G, k, host_grads=None, **over):
    from paper_2005_14038_b200 import hetpipe
    cid = hetpipe.comm_unique_id(lib)
    ctxs = [hetpipe.Context(hetpipe.config_from(cfg, world=G, rank=r, vw_span=k, **over), lib=lib)
            for r in range(G)]
    handles = [c.ipc_handle() for c in ctxs]
    out, errs = [None] * G, []

    def work(r):
        try:
            c = ctxs[r]
            c.connect(handles, cid)
            if host_grads is not None:
                c.schedule_set_host_grads(host_grads)
            c.run_schedule(cfg.tau, cfg.latency())
            with tempfile.NamedTemporaryFile(suffix=".trace") as f:
                tr = c.trace_lines(f.name)
            wg = c.read_weights(-1)
            m = c.read_weights(-2) if cfg.momentum else None
            wl = {v: c.read_weights(v) for v in range(cfg.num_vw) if c.local_len(v) or _has(cfg, G, k, v, r)}
            out[r] = (tr, wg, m, wl, c.stats())
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
    return out


def _has(cfg, G, k, v, r):
    return any((v * k + j) % G == r for j in range(k))


def check(cfg, G, k, out):
    o = run_schedule(cfg)
    for r in range(G):
        assert out[r][0] == o.trace, f"rank {r} trace"
    assert np.array_equal(np.concatenate([out[r][1] for r in range(G)]), o.wg)
    if cfg.momentum:
        assert np.array_equal(np.concatenate([out[r][2] for r in range(G)]), o.m)
    for v in range(cfg.num_vw):
        parts = [out[(v * k + j) % G][3][v] for j in range(k)]
        assert np.array_equal(np.concatenate(parts), o.wl[v]), f"w_local({v})"
    return o


CASES = [
    ("C3-G2", C3.replace(nparams=4099, waves=6), 2, 1),
    ("C3-G4", C3.replace(nparams=4099, waves=6), 4, 1),
    ("C3-G8", C3.replace(nparams=4099, waves=6), 8, 2),
    ("C5-G8", C5.replace(nparams=3001, waves=4, D=4), 8, 1),
    ("ED-G4", C3.replace(nparams=2048, waves=5, tau=(325,) * 4), 4, 4),
    ("N3-G4", WSPConfig("n3", 3, 2, 1, 999, 6, (3, 5, 4)), 4, 1),
    ("N2-G3-k2", WSPConfig("k2", 2, 3, 0, 777, 5, (4, 7)), 3, 2),
]


@pytest.mark.parametrize("name,cfg,G,k", CASES, ids=[c[0] for c in CASES])
def test_placement_matches_oracle(lib, name, cfg, G, k):
    out = run_placement(lib, cfg, G, k)
    check(cfg, G, k, out)
    nvl = sum(out[r][4].nvl_bytes for r in range(G))
    if k == G:
        assert nvl == 0          # ED-local: no exchange at all
    else:
        assert nvl > 0


@pytest.mark.parametrize("seed", range(24))
def test_placement_random(lib, seed):
    rng = random.Random(seed)
    G = rng.choice([2, 3, 4])
    k = rng.randint(1, G)
    N = rng.randint(1, 4)
    Nm = rng.randint(1, 4)
    tau = tuple(rng.randint(1, 9) for _ in range(N))
    mode = rng.choice([GRAD_FLOAT, GRAD_DYADIC])
    cfg = WSPConfig("rp", N, Nm, rng.randint(0, 3), rng.choice([64, 333, 1030, 4099]),
                    rng.randint(1, 6), tau, lr=0.01 if mode == GRAD_FLOAT else 2.0 ** -6,
                    momentum=rng.choice([0.0, 0.9]), grad_mode=mode,
                    pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
                    local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]),
                    lat=tuple(t * rng.randint(1, Nm + 1) for t in tau))
    out = run_placement(lib, cfg, G, k, merge_ticks=rng.randint(0, 1),
                        acc_slots=rng.choice([2, 3]), apply_mode=rng.randint(0, 1))
    check(cfg, G, k, out)


def rand_bounds(rng, P, G):
    inner = sorted(rng.sample(range(1, P // 32), G - 1))
    return [0] + [32 * x for x in inner] + [P]


@pytest.mark.parametrize("seed", range(10))
def test_uneven_ps_shards(lib, seed):
    """hp_config.ps_bounds: uneven PS shards (e.g. the paper's layer
    round-robin placement) change where each apply runs and what a
    pull reads, never the result."""
    rng = random.Random(500 + seed)
    G = rng.choice([2, 3, 4])
    k = rng.choice([1, G])
    N = rng.randint(1, 4)
    cfg = WSPConfig("ub", N, rng.randint(1, 3), rng.randint(0, 2), rng.choice([2048, 4099]),
                    rng.randint(2, 5), tuple(rng.randint(1, 9) for _ in range(N)),
                    momentum=rng.choice([0.0, 0.9]))
    b = rand_bounds(rng, cfg.nparams, G)
    out = run_placement(lib, cfg, G, k, ps_bounds=b)
    check(cfg, G, k, out)
    for r in range(G):
        assert len(out[r][1]) == b[r + 1] - b[r]


def test_layer_round_robin_bounds():
    from workloads import models as M
    b = M.layer_rr_bounds(M.vgg19(), 8)
    # fc6 (71.5% of VGG-19) makes one PS shard hold ~72% of the model
    # (the paper's default placement)
    assert abs((b[1] - b[0]) / b[-1] - 0.724) < 0.002
    assert b[-1] == 143_667_240 and all(x % 32 == 0 for x in b[1:-1])


def test_bad_ps_bounds(lib):
    from paper_2005_14038_b200 import hetpipe
    cfg = C3.replace(nparams=4099, waves=2)
    for bad in ([0, 100, 4099], [0, 4096, 4000], [1, 2048, 4099], [0, 2048, 4098]):
        with pytest.raises(hetpipe.HetPipeError):
            hetpipe.Context(hetpipe.config_from(cfg, world=2, rank=0, vw_span=1, ps_bounds=bad),
                            lib=lib)


def test_exchange_link_bytes_lockstep_peer(lib):
    """hp_profile_link: while every owner runs its apply launch of a lockstep
    batch (4 VWs, one per GPU, k = 1, equal speeds), each GPU's links carry in
    one direction the 3 remote u~ slices it loads plus the 3 owner-side pull
    stores it receives (or, out, the same from the other side): 6 x 4n bytes;
    the last round has no pull (Z16), so only the 3 loads."""
    from paper_2005_14038_b200 import hetpipe
    if os.environ.get("HP_PULL_PUSH") == "0":
        pytest.skip("reader-side pulls forced: other launch structure")
    G, P = 4, 4096
    cfg = WSPConfig("lk", G, 2, 0, P, 3, (5,) * G)
    cid = hetpipe.comm_unique_id(lib)
    ctxs = [hetpipe.Context(hetpipe.config_from(cfg, world=G, rank=r, vw_span=1), lib=lib)
            for r in range(G)]
    handles = [c.ipc_handle() for c in ctxs]
    links = [None] * G

    def work(r):
        c = ctxs[r]
        c.connect(handles, cid)
        c.profile_enable(True)
        c.run_schedule(cfg.tau, cfg.latency())
        links[r] = [x for x in c.profile_link() if x > 0]

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    n = P // G
    for r in range(G):
        assert links[r][:-1] == [6 * 4 * n] * (cfg.waves - 1), links[r]
        assert links[r][-1] == 3 * 4 * n
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("seed", range(24))
def test_placement_convex_and_update_frequency(lib, seed):
    """The weight-dependent CONVEX workload (NEXT-2) and F > 1 (NEXT-4) in the
    distributed placements: stash rings per VW stage, STASH ops after pulls and
    folds on every path (reader- and owner-side pulls), the F > 1 STRICT pull
    with its partial aggregate (reader-side), bit-exact against the oracle."""
    rng = random.Random(900 + seed)
    G = rng.choice([2, 3, 4])
    k = rng.randint(1, G)
    N = rng.randint(1, 4)
    Nm = rng.randint(1, 3)
    tau = tuple(rng.randint(1, 9) for _ in range(N))
    convex = seed % 2 == 0
    F = rng.choice([1, 2, 3]) if seed % 3 else 1
    cfg = WSPConfig("cf", N, Nm, rng.randint(0, 2), rng.choice([333, 1030, 4099]),
                    rng.randint(2, 4), tau, lr=0.05 if convex else 0.01,
                    momentum=rng.choice([0.0, 0.9]), grad_mode=3 if convex else GRAD_FLOAT,
                    pull_policy=rng.choice([PULL_EAGER, PULL_LAZY]),
                    local_semantics=rng.choice([LOCAL_STRICT, LOCAL_AT_LEAST]),
                    lat=tuple(t * rng.randint(1, Nm + 1) for t in tau), F=F)
    out = run_placement(lib, cfg, G, k, merge_ticks=rng.randint(0, 1),
                        apply_mode=rng.randint(0, 1))
    check(cfg, G, k, out)


@pytest.mark.parametrize("G,k", [(2, 1), (3, 2), (4, 1), (4, 4)])
def test_placement_external_host_gradients(lib, G, k):
    """EXTERNAL gradients in the distributed placements: every rank gets the
    VWs' whole host gradients and copies the stages it holds; the same Philox
    values as the synthetic mode give the oracle's arrays exactly."""
    from oracle import gradient
    cfg = C3.replace(nparams=2053, waves=3, D=1, tau=(3, 4, 6, 7))
    idx = np.arange(cfg.nparams)
    last_p = cfg.waves * cfg.Nm
    n = cfg.num_vw * last_p + 1
    bufs = [np.zeros(cfg.nparams, dtype=np.float32) for _ in range(n)]
    for v in range(cfg.num_vw):
        for p in range(1, last_p + 1):
            bufs[(v * last_p + p) % n][:] = gradient(idx, v, p, cfg)
    out = run_placement(lib, cfg, G, k, host_grads=bufs, grad_mode=GRAD_EXTERNAL)
    check(cfg, G, k, out)


def _fold_stream_launches(lib, cfg, G, k, **over):
    """Launches rank 0 issued on fold streams (HP_SPLIT_FOLDS: acc and folds
    in separate launches) over a whole schedule, via hp_profile_streams."""
    from paper_2005_14038_b200 import hetpipe
    cid = hetpipe.comm_unique_id(lib)
    ctxs = [hetpipe.Context(hetpipe.config_from(cfg, world=G, rank=r, vw_span=k, **over), lib=lib)
            for r in range(G)]
    handles = [c.ipc_handle() for c in ctxs]
    ids, errs = [None] * G, []

    def work(r):
        try:
            c = ctxs[r]
            c.connect(handles, cid)
            c.profile_enable(True)
            c.run_schedule(cfg.tau, cfg.latency())
            ids[r] = c.profile_streams()
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
    return int(np.sum(np.asarray(ids[0]) >= 3 + cfg.num_vw))


@pytest.mark.parametrize("conns,env,momentum,G,split", [
    ("32", {}, 0.0, 4, True),                       # C3 at 4 GPUs: one stage per GPU, SGD
    ("8", {}, 0.0, 4, False),                       # too few hardware queues
    (None, {}, 0.0, 4, False),                      # runtime default (8)
    ("32", {"HP_SPLIT_FOLDS": "0"}, 0.0, 4, False),  # explicit off
    ("32", {}, 0.9, 4, False),                      # heavy-ball momentum
    ("32", {}, 0.0, 2, False),                      # two VW stages per GPU
    ("8", {"HP_SPLIT_FOLDS": "1"}, 0.0, 2, True),   # explicit on
])
def test_split_folds_default_rule(lib, monkeypatch, conns, env, momentum, G, split):
    """The split acc / fold default (engine_dist.cpp finish_connect, DESIGN.md
    9h): on only for the peer exchange with SGD, at most one VW stage per GPU,
    a communicator and CUDA_DEVICE_MAX_CONNECTIONS >= 16; HP_SPLIT_FOLDS
    overrides. Parity of both forms: the placement cases above and
    tests/test_colocated_emu.py."""
    if conns is None:
        monkeypatch.delenv("CUDA_DEVICE_MAX_CONNECTIONS", raising=False)
    else:
        monkeypatch.setenv("CUDA_DEVICE_MAX_CONNECTIONS", conns)
    monkeypatch.delenv("HP_SPLIT_FOLDS", raising=False)
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    cfg = C3.replace(nparams=4096, waves=4, momentum=momentum)
    n = _fold_stream_launches(lib, cfg, G, 1)
    assert (n > 0) == split, n

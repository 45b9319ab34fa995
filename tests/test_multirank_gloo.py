"""The N>1 path on CPU: world_size 2 over gloo, each rank driving the real
engine (host-emulated device, tests/emu) on its ED-local shard. Checks that
every rank produces the identical trace, that the union of the shards equals
the oracle's full arrays, and that the max-over-ranks reduction the bench uses
works."""
import os
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import run_schedule
from workloads import C2, C3, WSPConfig


def _worker(rank, world, port, cfg, out_dir):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from emu import build_emu
    from paper_2005_14038_b200 import dist as hdist, hetpipe
    lib = hetpipe.load_test_library(build_emu.LIB)
    ctx = hdist.rank_context(cfg, rank, world, lib=lib)
    ctx.run_schedule(cfg.tau, cfg.latency())
    trace = ctx.trace_lines(os.path.join(out_dir, f"t{rank}.trace"))
    wg = ctx.read_weights(-1)
    wl = [ctx.read_weights(v) for v in range(cfg.num_vw)]
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    objs = [None] * world
    dist.all_gather_object(objs, (trace, wg, wl, float(t.item())))
    if rank == 0:
        np.save(os.path.join(out_dir, "ok.npy"), np.array([1]))
        import pickle
        with open(os.path.join(out_dir, "gathered.pkl"), "wb") as f:
            pickle.dump(objs, f)
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [C2.replace(nparams=4099, waves=4),
                                 C3.replace(nparams=1000, waves=6, momentum=0.9),
                                 WSPConfig("odd", 3, 2, 1, 97, 5, (3, 5, 4))],
                         ids=["C2", "C3-mom", "odd"])
def test_two_ranks_match_oracle(cfg):
    import pickle
    import socket
    from emu import build_emu
    build_emu.build()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, port, cfg, d), nprocs=2, join=True)
        with open(os.path.join(d, "gathered.pkl"), "rb") as f:
            objs = pickle.load(f)
    o = run_schedule(cfg)
    (t0, wg0, wl0, m0), (t1, wg1, wl1, m1) = objs
    assert t0 == t1 == o.trace
    assert m0 == m1 == 2.0
    assert np.array_equal(np.concatenate([wg0, wg1]), o.wg)
    for v in range(cfg.num_vw):
        assert np.array_equal(np.concatenate([wl0[v], wl1[v]]), o.wl[v])

"""Multi-GPU parity of the distributed placements (run under torchrun, one
rank per GPU; invoked by tests/test_gpu_multi.py). Every rank drives the real
library; rank 0 gathers the shards/stages and compares them with the oracle:
bit-exact arrays (the applies run in commit order) and identical traces.
Prints 'MULTI-GPU PARITY OK' on success, exits 1 otherwise."""
import os
import random
import sys

# as bench.py: enough hardware queues for the engine's streams (the library's
# split acc / fold default needs >= 16), before CUDA initialises
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch  # noqa: E402
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2005_14038_b200 import dist as hdist  # noqa: E402
from placement_check import check, collect, host_gradients  # noqa: E402
from workloads import (C3, C4, C5, C5E, GRAD_DYADIC, WSPConfig, ceil_shards,  # noqa: E402
                       sample_indices, even_shards)

from workloads import models as M  # noqa: E402

XPORT = {"peer": 0, "nccl": 1, "nvls": 2}


def run(cfg, G, k, rank, local, sampled, transport="peer", bounds=None, external=False):
    stream = torch.cuda.Stream(local)
    keep = None
    extra = {"ps_bounds": bounds} if bounds else {}
    if external:
        extra["grad_mode"] = 2
    if transport == "nvls":
        ctx, keep = hdist.symmetric_context(cfg, rank, G, k, device=local,
                                            stream=stream.cuda_stream, transport=XPORT["nvls"],
                                            **extra)
    else:
        ctx = hdist.placed_context(cfg, rank, G, k, device=local, stream=stream.cuda_stream,
                                   transport=XPORT[transport], **extra)
    if external:
        ctx.schedule_set_host_grads(host_gradients(cfg))
    ctx.run_schedule(cfg.tau, cfg.latency())
    res = collect(ctx, cfg, G, k, rank, sampled, bounds)
    ctx.close()
    del keep
    objs = [None] * G
    dist.all_gather_object(objs, res)
    return objs


def main():
    rank, G, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    # object exchange over gloo; the symmetric-memory rendezvous (NVLS) uses the
    # same group; the data itself moves over NVLink inside the library
    dist.init_process_group("cpu:gloo,cuda:nccl")
    lock = WSPConfig("lock", G, 4, 0, 40_000, 6, (7,) * G, lr=2.0 ** -6, grad_mode=GRAD_DYADIC)
    lockf = lock.replace(grad_mode=0, lr=0.01, nparams=40_003)
    c5e = C5E.replace(num_vw=G, tau=C5E.tau[:G], waves=3)
    # (cfg, k, sampled, transport, exact, lockstep batches expected)
    cases = [
        (C3.replace(nparams=40_000, waves=8), 1, None, "peer", True, False),
        (C3.replace(nparams=40_003, waves=8, momentum=0.9), max(1, G // 2), None, "peer", True, False),
        (WSPConfig("lazy", 3, 3, 1, 12_345, 7, (3, 5, 4), pull_policy=1, local_semantics=1), 1, None,
         "peer", True, False),
        (C4.replace(nparams=50_000, waves=4), G, None, "peer", True, False),
        (C5.replace(waves=2, D=4, num_vw=G, tau=C5.tau[:G]) if G <= 8 else None, 1, "sample",
         "peer", True, False),
        (C3.replace(waves=3), max(1, G // 4), "sample", "peer", True, False),
        # lockstep transports: DYADIC sums are exact in any order; FLOAT within Z15
        (lock, 1, None, "nccl", True, True),
        (lock, 1, None, "nvls", True, True),
        (lockf, 1, None, "nccl", False, True),
        (lockf, 1, None, "nvls", False, True),
        (c5e, 1, "sample", "nccl", False, True),
        (c5e, 1, "sample", "nvls", False, True),
        (c5e, 1, "sample", "peer", True, False),
        # EXTERNAL host gradients (the VWs' whole gradients, each rank copies its stages)
        (C3.replace(nparams=20_000, waves=4, D=1), 1, None, "peer", True, False, "external"),
        (C3.replace(nparams=20_000, waves=4), max(1, G // 2), None, "peer", True, False, "external"),
        # the paper's default layer round-robin PS placement: uneven shards
        (c5e, 1, "sample", "nvls", False, True, "layer_rr"),
        (C5.replace(waves=2, D=4, num_vw=G, tau=C5.tau[:G]), 1, "sample", "peer", True, False,
         "layer_rr"),
        # never lockstep (heavy-ball momentum is per push, Z11): the NVLS and NCCL
        # contexts take the PEER path for every batch, bit-exact
        (C5.replace(waves=3, D=4, num_vw=G, tau=C5.tau[:G], nparams=40_000), 1, None, "nvls",
         True, False),
        (C5.replace(waves=3, D=4, num_vw=G, tau=C5.tau[:G], nparams=40_000), 1, None, "nccl",
         True, False),
    ]
    # randomized placements (the stream / event / barrier logic on real GPUs):
    # same seeds on every rank, so every rank builds the same list
    rng = random.Random(int(os.environ.get("HP_MULTI_SEED", "2005")))
    for _ in range(int(os.environ.get("HP_MULTI_RANDOM", "16"))):
        N = rng.randint(1, 8)
        Nm = rng.randint(1, 4)
        tau = tuple(rng.randint(1, 9) for _ in range(N))
        k = rng.randint(1, G)
        convex = rng.random() < 0.3
        cfg = WSPConfig("rnd", N, Nm, rng.randint(0, 3), rng.choice([4099, 20_000, 33_333]),
                        rng.randint(2, 6), tau, momentum=rng.choice([0.0, 0.9]),
                        pull_policy=rng.choice([0, 1]), local_semantics=rng.choice([0, 1]),
                        lat=tuple(t * rng.randint(1, Nm + 1) for t in tau),
                        grad_mode=3 if convex else 0, lr=0.05 if convex else 0.01,
                        F=rng.choice([1, 1, 2]))
        cases.append((cfg, k, None, rng.choice(["peer", "peer", "nccl"]), None, None))
    ok = True
    for case in cases:
        cfg, k, mode, xport, exact, want_lock = case[:6]
        if cfg is None:
            continue
        external = len(case) > 6 and case[6] == "external"
        bounds = (M.layer_rr_bounds(M.vgg19(), G) if len(case) > 6 and case[6] == "layer_rr" else
                  ceil_shards(cfg.nparams, G) if xport == "nccl" and k == 1 else None)
        sampled = (sample_indices(cfg.nparams, 104729, bounds or even_shards(cfg.nparams, G))
                   if mode else None)
        objs = run(cfg, G, k, rank, local, sampled, xport, bounds, external)
        if rank == 0:
            try:
                nlock = objs[0][5]
                if exact is None:            # random case: exact unless a lockstep batch ran
                    exact, want_lock = nlock == 0 or cfg.grad_mode == GRAD_DYADIC, nlock > 0
                check(cfg, G, k, objs, sampled, exact)
                assert (nlock > 0) == want_lock, f"lockstep batches {nlock}"
                print(f"ok {cfg.name} N={cfg.num_vw} P={cfg.nparams} G={G} k={k} {xport} "
                      f"lockstep={nlock}", flush=True)
            except AssertionError as e:
                ok = False
                print(f"FAIL {cfg.name} G={G} k={k} {xport}: {e}", flush=True)
        dist.barrier()
    if rank == 0:
        print("MULTI-GPU PARITY OK" if ok else "MULTI-GPU PARITY FAILED", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

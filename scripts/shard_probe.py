"""Per-rank cost of the ED-local placement at world size W, measured on ONE
GPU: rank 0's shard (P/W params of every VW and of the PS) driven by the same
controller (each ED-local rank is independent), so the
per-rank step time at W = 8 can be seen on a single B200.

    python scripts/shard_probe.py --world 8 [--config C2] [--steps 100]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2005_14038_b200 import dist as hdist  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    run = cfg.replace(waves=args.warmup + args.steps + 2)
    N = cfg.num_vw
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    out = {}
    for pdl in (os.environ.get("HP_PDL", "1"),):
        ctx = hdist.rank_context(run, 0, args.world, device=0, stream=stream.cuda_stream)
        ctx.trace_enable(False)
        ctx.schedule_begin(run.tau, run.latency())
        ctx.schedule_advance(N * args.warmup)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0 = ctx.stats()
        e0.record(stream)
        for k in range(args.steps):
            ctx.schedule_advance(N * (args.warmup + k + 1))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        s1 = ctx.stats()
        gbs = (s1.alg_bytes - s0.alg_bytes) / args.steps / (ms / 1e3) / 1e9
        out[f"pdl{pdl}"] = {"ms_per_step": ms, "alg_GBps": gbs,
                            "launches_per_step": (s1.launches - s0.launches) / args.steps}
        ctx.close()
    print(json.dumps({"config": cfg.name, "world": args.world, **out}))


if __name__ == "__main__":
    main()

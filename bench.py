#!/usr/bin/env python
"""Benchmark of the WSP synchronization hot path (HetPipe, arXiv 2005.14038).

Metric (BASELINE.json): synced params/sec (and wave-sync latency) vs the
HBM roofline. A STEP is one WSP round of the deterministic schedule: every VW
completes one wave of N_m minibatches (accumulate + fold), pushes it, the PS
applies it and the VW pulls under the staleness bound D -- all of SURVEY.md
8(a) rows a1-a8 -- i.e. the controller advances until N more pushes are
committed. value = pushes committed in the timed region x P / device time.

Workload at N=1: BASELINE.json configs[1] = C2, 4 VWs with Node-Partition
speeds, N_m=4, D=0, 60,192,808 params (ResNet-152 size), FLOAT synthetic
gradients (Philox). At N>1 the same model is sharded ED-local over the ranks
(each rank owns P/N params of every VW and the PS shard; no exchange exists,
PAPER.md P:104-106), so scaling is STRONG (fixed model).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hetpipe|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from workloads import CONFIGS, GRAD_EXTERNAL, PMP_SOURCE  # noqa: E402

METRIC = "synced params/sec"
UNIT = "params/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(cfg_name):
    """dram read+write bytes per launch of the dominant kernel from the committed
    `ncu --set full` summary (profiles/ncu_summary.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get("traffic_bytes_per_launch", {}).get(cfg_name)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sms, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9 or parts[1] != str(self.index):
                continue
            try:
                sms.append(float(parts[2]))
                mx.append(float(parts[3]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sms)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _oracle_chunk(job):
    """One worker of the all-cores oracle timing: the oracle as it stands on the
    param range [lo, hi) of the schedule (every op is element-wise in the param
    index, SURVEY.md 8(c) "sampled parity", so ranges are independent)."""
    import numpy as np
    from oracle import run_schedule
    cfg, lo, hi = job
    t0 = time.time()
    o = run_schedule(cfg, idx=np.arange(lo, hi))
    return t0, time.time(), len(o.commit) if hasattr(o, "commit") else None


def cpu_baseline(cfg, params=1 << 21, rounds=4, per_core=1 << 20, max_cores=64):
    """The oracle as it stands (numpy) on a bounded sample of the same workload:
    (1) one thread over the first `params` params of the schedule for `rounds`
    rounds; (2) every host core, each process running the oracle on its own
    `per_core`-param range of the same schedule. Returns synced params/s."""
    import multiprocessing as mp

    import numpy as np
    from oracle import run_schedule
    c = cfg.replace(waves=rounds)
    marks = []
    t0 = time.perf_counter()
    run_schedule(c, idx=np.arange(min(params, c.nparams)),
                 on_tick=lambda t, sm: marks.append((time.perf_counter(), len(sm.commit))))
    dt = time.perf_counter() - t0
    commits = marks[-1][1]
    one = commits * min(params, c.nparams) / dt
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    cores = max(1, min(cores, max_cores, c.nparams // per_core or 1))
    jobs = [(c, k * per_core, min((k + 1) * per_core, c.nparams)) for k in range(cores)]
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_chunk, jobs)
    span = max(r[1] for r in res) - min(r[0] for r in res)
    allc = commits * sum(hi - lo for _, lo, hi in jobs) / span
    return {"value": allc, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1core": one,
            "sample": f"{cfg.name} schedule, {rounds} rounds ({commits} pushes): all-cores = "
                      f"{cores} processes x {per_core} params each ({span:.1f} s wall); "
                      f"1 core = params [0,{min(params, c.nparams)}) ({dt:.1f} s), numpy"}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle timed on the host, each step one WSP
    round of the same schedule over a bounded param sample."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import numpy as np
    from oracle import run_schedule
    sample = args.ref_params
    c = cfg.replace(waves=args.warmup + args.steps + 1)
    N = c.num_vw
    marks = {}
    t_start = [None]

    def on_tick(t, sm):
        k = len(sm.commit)
        if k >= N * args.warmup and t_start[0] is None:
            t_start[0] = (time.perf_counter(), k)
        if k >= N * (args.warmup + args.steps) and "end" not in marks:
            marks["end"] = (time.perf_counter(), k)
            raise StopIteration

    try:
        run_schedule(c, idx=np.arange(sample), on_tick=on_tick)
    except StopIteration:
        pass
    (t0, k0), (t1, k1) = t_start[0], marks["end"]
    dt = t1 - t0
    value = (k1 - k0) * sample / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "num_vw": N, "Nm": c.Nm, "D": c.D,
                   "nparams": c.nparams, "sample_params": sample, "tau": list(c.tau)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {sample} params of {cfg.name}, one WSP round per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hetpipe", choices=["hetpipe", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--profile-steps", type=int, default=20,
                    help="steps of the separate per-launch-profiled pass after the timed region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-params", type=int, default=1 << 18)
    ap.add_argument("--merge-ticks", type=int, default=1)
    ap.add_argument("--apply-mode", type=int, default=0,
                    help="0: defer PS applies to the observing pull; 1: apply on arrival")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl", "nvls"],
                    help="exchange of lockstep batches (distributed placements; include/hetpipe.h "
                         "HP_XPORT_*): peer = fused NVLink loads, nccl = reduce-scatter/all-gather "
                         "baseline, nvls = multimem through the NVSwitch")
    ap.add_argument("--timing", default="proxy", choices=["proxy", "pmp"],
                    help="per-VW tau/L: the speed proxy (reading Z14) or derived from "
                         "partitioning the model over each VW's GPUs and simulating its "
                         "pipeline (hp_partition + hp_pipeline_tau_latency, NEXT-1)")
    ap.add_argument("--ps", default="even", choices=["even", "layer_rr"],
                    help="PS shard boundaries of the distributed placements: even (reading Z12) "
                         "or the paper's default layer round-robin (P:100-103) on the config's "
                         "model (uneven shards; hp_config.ps_bounds)")
    ap.add_argument("--grad", default="float", choices=["float", "convex"],
                    help="synthetic gradient: weight-independent Philox FLOAT draws, or the "
                         "weight-dependent CONVEX workload (NEXT-2: every gradient reads the "
                         "w_local its minibatch saw at START, kept in a stash ring)")
    ap.add_argument("--pull", default="eager", choices=["eager", "lazy"],
                    help="pull policy (reading Z6): every gate pulls, or only when the held "
                         "version is older than the bound needs (P:932)")
    ap.add_argument("--D", type=int, default=-1,
                    help="override the config's clock-distance threshold D (C5's sweep: 0, 4, 32)")
    ap.add_argument("--update-freq", type=int, default=1,
                    help="F (NEXT-4): one clock = F waves; a step is still one WSP round "
                         "(N pushes), each push carrying F*Nm minibatches")
    ap.add_argument("--num-vw", type=int, default=0,
                    help="override the config's VW count (C5E defaults to one VW per GPU)")
    ap.add_argument("--span", type=int, default=0,
                    help="N>1: GPUs per VW of the distributed placement (k<N exchanges over "
                         "NVLink); 0 = ED-local shards (no exchange)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    nvw = args.num_vw or (int(os.environ.get("WORLD_SIZE", "1")) if cfg.name in ("C5E", "HVD")
                          else 0)
    if nvw:
        cfg = cfg.replace(num_vw=nvw, tau=tuple((list(cfg.tau) * 8)[:nvw]))
    if args.update_freq > 1:
        cfg = cfg.replace(F=args.update_freq)
    if args.D >= 0:
        cfg = cfg.replace(D=args.D)
    if args.pull == "lazy":
        cfg = cfg.replace(pull_policy=1)
    if args.grad == "convex":
        from workloads import GRAD_CONVEX
        cfg = cfg.replace(grad_mode=GRAD_CONVEX)
    if args.timing == "pmp":
        from paper_2005_14038_b200 import schedule
        model, vws = PMP_SOURCE[cfg.name]
        tau, lat = schedule.policy_timing(model, "", cfg.Nm, vws[:cfg.num_vw])
        cfg = cfg.replace(tau=tau, lat=lat)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_14038_b200 import dist as hdist

    ws, rank, local = _dist()
    if ws != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
    torch.cuda.set_device(local)
    if ws > 1:
        # libraries print to fd 1 (NCCL's version banner): send C-level stdout to
        # stderr and keep the real stdout for the one JSON line
        real_out = os.dup(1)
        os.dup2(2, 1)
        sys.stdout = os.fdopen(real_out, "w")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if ws > 1:
            dist.barrier()

    lo, hi = hdist.shard_bounds(cfg.nparams, ws, rank)
    N = cfg.num_vw
    prof_steps = max(1, min(args.steps, args.profile_steps))
    waves = args.warmup + args.steps + prof_steps + 2
    run_cfg = cfg.replace(waves=waves)
    stream = torch.cuda.Stream(local)          # a real stream: the library launches on it
    torch.cuda.set_stream(stream)              # and the timing events below record on it
    placed = ws > 1 and args.span > 0
    keep = None
    xport = {"peer": 0, "nccl": 1, "nvls": 2}[args.transport]
    extra = {}
    if placed and args.ps == "layer_rr":
        from workloads import models as wm
        extra["ps_bounds"] = wm.layer_rr_bounds(wm.MODELS[PMP_SOURCE[cfg.name][0]](), ws)
    if placed and args.transport == "nvls":
        ctx, keep = hdist.symmetric_context(run_cfg, rank, ws, args.span, device=local,
                                            stream=stream.cuda_stream, merge_ticks=args.merge_ticks,
                                            apply_mode=args.apply_mode, transport=xport, **extra)
    elif placed:
        ctx = hdist.placed_context(run_cfg, rank, ws, args.span, device=local,
                                   stream=stream.cuda_stream, merge_ticks=args.merge_ticks,
                                   apply_mode=args.apply_mode, transport=xport, **extra)
    else:
        ctx = hdist.rank_context(run_cfg, rank, ws, device=local, stream=stream.cuda_stream,
                                 merge_ticks=args.merge_ticks, apply_mode=args.apply_mode)
    ctx.trace_enable(False)
    from paper_2005_14038_b200 import hetpipe as _hp
    arena = _hp.arena_bytes(ctx.cfg)       # device bytes this rank's context holds
    ctx.schedule_begin(run_cfg.tau, run_cfg.latency())
    sampler = ClockSampler(local)
    ctx.schedule_advance(N * args.warmup)
    torch.cuda.synchronize()
    barrier()
    st0 = ctx.stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    # ---- timed region: K steps, no per-launch instrumentation
    ev0.record(stream)
    for k in range(args.steps):
        ctx.schedule_advance(N * (args.warmup + k + 1))
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms_timed = ev0.elapsed_time(ev1)
    st1 = ctx.stats()
    # ---- profiled pass over the next steps of the same schedule: per-launch
    # CUDA events on the launch streams (roofline, launch mix, sync latency)
    ctx.profile_enable(True)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    pe0.record(stream)
    for k in range(prof_steps):
        ctx.schedule_advance(N * (args.warmup + args.steps + k + 1))
    pe1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = pe0.elapsed_time(pe1)
    kern_ms, kern_bytes, kern_launches = ctx.profile_read()
    l_ms, l_bytes, l_shape, l_sync, l_t0 = ctx.profile_launches()
    # device time during which at least one tick kernel runs (union of the
    # launch intervals: the distributed placements launch on several streams)
    busy_ms, cur_a, cur_b = 0.0, None, None
    for a, d in sorted((float(t0), float(t)) for t0, t, by in zip(l_t0, l_ms, l_bytes)
                       if by > 0):      # barriers (0 bytes) are not kernel time
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                busy_ms += cur_b - cur_a
            cur_a, cur_b = a, a + d
        else:
            cur_b = max(cur_b, a + d)
    if cur_b is not None:
        busy_ms += cur_b - cur_a
    # sync-only time: each launch's device time attributed to synchronisation
    # in proportion to its sync share of the algorithmic bytes (the push/apply/
    # pull ops are fused with accumulation, so they have no launch of their own)
    sync_ms = float(sum(float(t) * float(sy) / float(by)
                        for t, by, sy in zip(l_ms, l_bytes, l_sync) if by > 0))
    s_ms, s_vw, s_waited = ctx.profile_sync_latency()
    l_link = ctx.profile_link()
    xl = [(float(t), float(b)) for t, b in zip(l_ms, l_link) if b > 0]
    xch = None
    if xl:
        xt, xb = sum(t for t, _ in xl), sum(b for _, b in xl)
        xch = {"launches": len(xl), "ms": xt, "link_bytes": xb,
               "achieved_GBps": xb / (xt / 1e3) / 1e9, "peak_GBps": 770.0,
               "frac": xb / (xt / 1e3) / 1e9 / 770.0, "bound": "nvlink",
               "frac_vs_nominal_900": xb / (xt / 1e3) / 1e9 / 900.0,
               "def": "exchange launches only (peer loads/stores, NVLS multimem, NCCL "
                      "collectives): algorithmic NVLink bytes per direction / their device "
                      "time, rank 0; peak = guide-measured peer copy per direction"}
    sync_us = [1e3 * float(x) for x in s_ms]
    sync_unblocked = [1e3 * float(x) for x, w in zip(s_ms, s_waited) if not w]
    mix = {}
    for t_ms, by, sh in zip(l_ms, l_bytes, l_shape):
        sh = int(sh) & 0xFFFFFFFF
        key = (f"c{sh & 15}i{(sh >> 4) & 15}a{(sh >> 8) & 255}g{(sh >> 16) & 255}"
               f"f{(sh >> 24) & 127}")
        if (sh >> 24) & 127 == 127:
            key = "nccl_reduce_scatter" if (sh >> 8) & 255 else "nccl_all_gather"
        elif (sh >> 24) & 127 == 126:
            key = "barrier"
        e = mix.setdefault(key, [0, 0.0, 0.0])
        e[0] += 1
        e[1] += float(t_ms)
        e[2] += float(by)
    launch_mix = {k: {"n": n, "us_mean": 1e3 * t / n, "GBps": b / (t / 1e3) / 1e9}
                  for k, (n, t, b) in sorted(mix.items(), key=lambda kv: -kv[1][1])}
    st2 = ctx.stats()
    commits = st1.commits - st0.commits
    pcommits = st2.commits - st1.commits
    t = torch.tensor([ms_timed, sync_ms * commits / max(pcommits, 1)], dtype=torch.float64,
                     device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0].item())
    sync_ms_max = float(t[1].item())     # scaled from the profiled pass to K steps
    value = commits * cfg.nparams / (ms_max / 1e3)
    launches = st1.launches - st0.launches
    nvl = torch.tensor([st1.nvl_bytes - st0.nvl_bytes], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(nvl, op=dist.ReduceOp.MAX)
    nvl_bytes_max = float(nvl.item())
    sync_waits = [int(x) for x in st1.wait_ticks[:N]]
    lock_batches = st1.lockstep_batches - st0.lockstep_batches
    ctx.close()
    del ctx, keep
    torch.cuda.empty_cache()

    # ---------------- e2e: host gradients in, w_global out, through the C-ABI
    e2e = None
    if not args.no_e2e and cfg.grad_mode != 3:
        e_steps = max(1, args.e2e_steps)
        ecfg = cfg.replace(waves=3 + e_steps + 1)
        # host gradients: single-rank contexts take their shard, the distributed
        # placements each VW's whole gradient (every rank copies its stages)
        nloc = cfg.nparams if placed else hi - lo
        host = [torch.empty(nloc, dtype=torch.float32, pin_memory=True) for _ in range(4)]
        rng = np.random.default_rng(cfg.seed)
        for h in host:
            h.numpy()[:] = (rng.random(nloc, dtype=np.float32) - np.float32(0.5))
        ekeep = None
        if placed and args.transport == "nvls":
            ectx, ekeep = hdist.symmetric_context(ecfg, rank, ws, args.span, device=local,
                                                  stream=stream.cuda_stream, transport=xport,
                                                  grad_mode=GRAD_EXTERNAL, **extra)
        elif placed:
            ectx = hdist.placed_context(ecfg, rank, ws, args.span, device=local,
                                        stream=stream.cuda_stream, transport=xport,
                                        grad_mode=GRAD_EXTERNAL, **extra)
        else:
            ectx = hdist.rank_context(ecfg, rank, ws, device=local, stream=stream.cuda_stream,
                                      grad_mode=GRAD_EXTERNAL)
        out = torch.empty(max(1, ectx.local_len(-1)), dtype=torch.float32, pin_memory=True)
        ectx.trace_enable(False)
        ectx.schedule_set_host_grads([h.numpy() for h in host])
        ectx.schedule_begin(ecfg.tau, ecfg.latency())
        ectx.schedule_advance(N * 3)
        ectx.read_weights(-1, out=out.numpy())
        torch.cuda.synchronize()
        barrier()
        s0 = ectx.stats()
        t0 = time.perf_counter()
        for k in range(e_steps):
            ectx.schedule_advance(N * (3 + k + 1))
            ectx.read_weights(-1, out=out.numpy())      # D2H of the step's result
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        s1 = ectx.stats()
        tt = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
        if ws > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        ecommits = s1.commits - s0.commits
        completes_per_step = N * cfg.Nm
        # every minibatch's gradient crosses PCIe once in total (a rank copies its
        # shard / its stages of it); w_global is read back once across the ranks
        e2e = {"value": ecommits * cfg.nparams / dt, "unit": UNIT,
               "h2d_bytes_per_step": completes_per_step * cfg.nparams * 4,
               "d2h_bytes_per_step": cfg.nparams * 4,
               "steps": e_steps, "ms_per_step": 1e3 * dt / e_steps,
               "path": "hp_schedule_set_host_grads + hp_schedule_advance + hp_read_weights(-1)"}
        ectx.close()
        del ekeep

    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_kind = _peaks()
    # algorithmic bytes over the time some tick kernel is running (= the sum of
    # launch durations on one stream; the union of intervals across streams)
    achieved = kern_bytes / (busy_ms / 1e3) / 1e9 if busy_ms > 0 else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "num_vw": N, "Nm": cfg.Nm, "D": cfg.D, "F": cfg.F,
                   "nparams": cfg.nparams, "tau": list(cfg.tau),
                   "lat": list(cfg.latency()), "timing": args.timing, "placement":
                   (f"distributed, {args.span} GPU(s) per VW, PS sharded over {ws}" if placed
                    else "ED-local shards" if ws > 1 else "single GPU"),
                   "grad": ("CONVEX a(w_p - b) + sigma xi, w_p from the START stash"
                            if args.grad == "convex" else "Philox FLOAT in-kernel"),
                   "pull": args.pull.upper(), "local": "STRICT",
                   "apply": "on arrival" if args.apply_mode else "deferred to the observing pull",
                   "transport": args.transport if placed else None,
                   "ps_shards": args.ps if placed else None,
                   "lockstep_batches": lock_batches if placed else None,
                   "l2": "inputs larger than L2 (>= 13 x 230 MiB buffers per GPU)",
                   "arena_GiB_per_rank": arena / 2 ** 30},
        "images_per_sec_equiv": commits * 32 * cfg.Nm * cfg.F / (ms_max / 1e3),
        "sync_only": ({"value": commits * cfg.nparams / (sync_ms_max / 1e3), "unit": UNIT,
                       "ms_per_step": sync_ms_max / args.steps,
                       "def": "push+apply+pull only: each launch's device time attributed to "
                              "synchronisation by its share of algorithmic bytes (w_global/m, "
                              "u~ reads, pull writes); max over ranks"}
                      if sync_ms_max > 0 else None),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _ncu_traffic(cfg.name),
                     "frac_vs_nominal_8000": achieved / 8000.0,
                     "peak_kind": peak_kind, "kernel": "hp::tick_kernel (all launches)",
                     "kernel_ms": kern_ms, "busy_ms": busy_ms, "launches": kern_launches,
                     "alg_bytes_per_launch": kern_bytes / max(kern_launches, 1)},
        "exchange_roofline": xch,
        "nvlink": {"bytes_per_step_max_rank": nvl_bytes_max / args.steps,
                   "GBps_over_step": nvl_bytes_max / (ms_max / 1e3) / 1e9,
                   "peak_GBps": 770.0, "peak_kind": "guide-measured peer copy per direction"},
        "wave_sync_latency_us": (
            {"p50": float(np.percentile(sync_us, 50)), "p99": float(np.percentile(sync_us, 99)),
             "max": float(np.max(sync_us)), "n": len(sync_us),
             "unblocked": ({"p50": float(np.percentile(sync_unblocked, 50)),
                            "p99": float(np.percentile(sync_unblocked, 99)),
                            "n": len(sync_unblocked)} if sync_unblocked else None),
             "def": "per (VW, wave), rank 0: device time from the start of the launch carrying "
                    "the VW's wave-end COMPLETE (u~ final = push) to the end of the launch that "
                    "wrote its pulled w_local (hp_profile_sync_latency); all records include gate "
                    "waits, `unblocked` only those whose VW did not wait"}
            if sync_us else None),
        "kernel_share_of_step": busy_ms / ms if ms > 0 else None,
        "launch_mix": launch_mix,
        "gpu_launches": launches,
        "clocks": clocks,
        "wait_ticks_per_vw": sync_waits,
        "e2e": e2e,
    }
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

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
gradients (Philox). At N>1: configs[2] = C3 (Hybrid-Distribution speeds, D=4,
the same model) with the PS sharded over the N GPUs and SURVEY.md 8(d)'s
placement (one replica per VW at 2 and 4 GPUs, two-stage VWs at 8): pushes and
pulls cross NVLink inside the tick kernels. Scaling is STRONG (fixed model).
The N>1 line also carries the ED-local C2 placement (no exchange)
and the same config on one GPU.

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

# hardware work queues per CUDA context, read once at context creation (before
# torch initialises CUDA): the distributed engine runs the exchange, the
# accumulation and the fold launches on separate streams, which the default 8
# queues alias (the library's split acc / fold default asks for
# >= 16, include/hetpipe.h hp_connect)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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
            "value_1core": one, "cpu_model": cpu_model(),
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
                         "cpu_model": cpu_model(),
                         "sample": f"first {sample} params of {cfg.name}, one WSP round per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# SURVEY.md 8(d) placements of the multi-GPU configs: GPUs per VW (k) at G GPUs.
# C3 (BASELINE configs[2]): G=2 and G=4 one replica per VW (k=1), G=8 two-stage
# VWs (k=2); C5 / C5E / HVD: one VW per GPU (k=1); C2 / C4: ED-local shards
# (every VW spans every GPU, stage q = PS shard q: no exchange).
AUTO_SPAN = {"C3": {2: 1, 4: 1, 8: 2}, "C5": 1, "C5E": 1, "HVD": 1}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def nvlink_peak():
    """Per-direction NVLink peak: the on-box measurement of scripts/nvlink_peak.py
    (profiles/nvlink_peak.json), else the profiling guide's peer-copy figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "nvlink_peak.json")) as f:
            pk = json.load(f)
        return float(pk["peer_copy_GBps_per_direction"]), "measured on-box (profiles/nvlink_peak.json)"
    except Exception:
        return 770.0, "guide-measured peer copy per direction (fallback)"


class NvlinkCounters:
    """NVLink data bytes this GPU transmitted / received, from NVML's per-link
    counters (nvmlDeviceGetFieldValues: NVLINK_THROUGHPUT_DATA_TX / _RX, KiB,
    one value per link), read around the timed region."""
    FIELDS = ((138, 139, 1024.0, "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB)"),
              (202, 204, 1.0, "NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES"))

    def __init__(self, index):
        self.ok, self.field = False, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.links = []
            for link in range(18):
                try:
                    if pynvml.nvmlDeviceGetNvLinkState(self.h, link):
                        self.links.append(link)
                except Exception:
                    continue
            for tx, rx, scale, name in self.FIELDS:
                try:
                    self._read(tx, rx, scale)
                    self.tx, self.rx, self.scale, self.field = tx, rx, scale, name
                    self.ok = True
                    break
                except Exception:
                    continue
        except Exception:
            self.ok = False

    def _read(self, tx, rx, scale):
        req = [(tx, ln) for ln in self.links] + [(rx, ln) for ln in self.links]
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, req)
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError("field not supported")
            out.append(float(v.value.ullVal) * scale)
        n = len(self.links)
        return sum(out[:n]), sum(out[n:])

    def read(self):
        if not self.ok:
            return None
        try:
            return self._read(self.tx, self.rx, self.scale)
        except Exception:
            return None


def resolve_config(args, ws):
    name = args.config or ("C2" if ws == 1 else "C3")
    cfg = CONFIGS[name]
    span = args.span
    if span < 0:                       # auto: SURVEY.md 8(d) placement
        a = AUTO_SPAN.get(name, 0)
        span = (a.get(ws, 1) if isinstance(a, dict) else a) if ws > 1 else 0
    nvw = args.num_vw or (ws if name in ("C5E", "HVD") and ws > 1 else 0)
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
    return cfg, span


def survey_bytes_per_param(pushes, apply_batches, cfg):
    """SURVEY.md 8(d) algorithmic bytes per parameter: per VW-wave 16*U
    (accumulate 16U-12 incl. the fold a pull overwrites, + 4 read of u~ at the
    PS + 4+4 pull), per apply batch 8 (w_global RMW; +8 momentum), U = F*Nm
    minibatches per push. Defined for the synthetic gradients (FLOAT/DYADIC)."""
    U = cfg.F * cfg.Nm
    return 16.0 * U * pushes + 8.0 * (2 if cfg.momentum else 1) * apply_batches


class Run:
    """Device context(s) of one measured configuration on this rank."""

    def __init__(self, cfg, span, args, ws, rank, local, stream, extra, **over):
        from paper_2005_14038_b200 import dist as hdist
        self.keep = None
        xport = {"peer": 0, "nccl": 1, "nvls": 2}[args.transport]
        self.placed = ws > 1 and span > 0
        kw = dict(merge_ticks=args.merge_ticks, apply_mode=args.apply_mode,
                  acc_slots=args.acc_slots)
        kw.update(over)
        if self.placed and args.transport == "nvls":
            self.ctx, self.keep = hdist.symmetric_context(cfg, rank, ws, span, device=local,
                                                          stream=stream.cuda_stream,
                                                          transport=xport, **extra, **kw)
        elif self.placed:
            self.ctx = hdist.placed_context(cfg, rank, ws, span, device=local,
                                            stream=stream.cuda_stream, transport=xport,
                                            **extra, **kw)
        else:
            self.ctx = hdist.rank_context(cfg, rank, ws, device=local, stream=stream.cuda_stream,
                                          **kw)

    def close(self):
        self.ctx.close()
        self.ctx = None
        self.keep = None


def measure(cfg, span, args, ws, rank, local, stream, steps, warmup, profile_steps, graph,
            extra, sampler=False, nvml=None):
    """Warm up, then time exactly `steps` WSP rounds on the device (CUDA events
    on the launch stream, barrier + synchronize on both sides, max over ranks),
    then an optional per-launch-profiled pass over the next rounds."""
    import torch
    import torch.distributed as dist

    def barrier():
        if ws > 1:
            dist.barrier()

    N = cfg.num_vw
    run_cfg = cfg.replace(waves=warmup + steps + profile_steps + 2)
    run = Run(run_cfg, span, args, ws, rank, local, stream, extra)
    ctx = run.ctx
    ctx.trace_enable(False)
    from paper_2005_14038_b200 import hetpipe as _hp
    arena = _hp.arena_bytes(ctx.cfg)
    ctx.schedule_begin(run_cfg.tau, run_cfg.latency())
    if graph:
        g = ctx.schedule_capture(N * warmup)
        g.launch()
        g.close()
    else:
        ctx.schedule_advance(N * warmup)
        ctx.flush()
    torch.cuda.synchronize()
    barrier()
    st0 = ctx.stats()
    g = ctx.schedule_capture(N * (warmup + steps)) if graph else None   # host work now
    clk = ClockSampler(local) if sampler else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    n0 = nvml.read() if nvml else None
    # ---- timed region: `steps` WSP rounds, no per-launch instrumentation
    ev0.record(stream)
    if graph:
        g.launch()
    else:
        for k in range(steps):
            ctx.schedule_advance(N * (warmup + k + 1))
        ctx.flush()                  # join the side streams before the end event
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    n1 = nvml.read() if nvml else None
    clocks = clk.stop() if clk else None
    if g is not None:
        g.close()
    ms_timed = ev0.elapsed_time(ev1)
    st1 = ctx.stats()
    res = {"ms_timed": ms_timed, "commits": st1.commits - st0.commits,
           "alg_bytes": st1.alg_bytes - st0.alg_bytes, "launches": st1.launches - st0.launches,
           "ticks": st1.ticks - st0.ticks, "apply_batches": st1.apply_batches - st0.apply_batches,
           "nvl_alg": st1.nvl_bytes - st0.nvl_bytes,
           "lockstep": st1.lockstep_batches - st0.lockstep_batches,
           "waits": [int(x) for x in st1.wait_ticks[:min(N, 8)]], "clocks": clocks,
           "arena": arena, "placed": run.placed,
           "nvml": (None if n0 is None or n1 is None else
                    {"tx_bytes": n1[0] - n0[0], "rx_bytes": n1[1] - n0[1], "field": nvml.field})}
    if profile_steps > 0:
        res.update(profiled_pass(ctx, N, warmup + steps, profile_steps, stream, barrier))
    t = torch.tensor([ms_timed, res.get("sync_ms", 0.0) * res["commits"] /
                      max(res.get("pcommits", 1), 1)], dtype=torch.float64,
                     device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res["ms_max"] = float(t[0].item())
    res["sync_ms_max"] = float(t[1].item())
    res["value"] = res["commits"] * cfg.nparams / (res["ms_max"] / 1e3)
    run.close()
    torch.cuda.empty_cache()
    return res


def profiled_pass(ctx, N, done_steps, prof_steps, stream, barrier):
    """Per-launch CUDA events over the next rounds of the same schedule: launch
    mix, union of the launch intervals, byte-attributed sync time, wave-sync
    latency, exchange bytes."""
    import torch
    st0 = ctx.stats()
    ctx.profile_enable(True)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    pe0.record(stream)
    for k in range(prof_steps):
        ctx.schedule_advance(N * (done_steps + k + 1))
    ctx.flush()
    pe1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = pe0.elapsed_time(pe1)
    kern_ms, kern_bytes, kern_launches = ctx.profile_read()
    l_ms, l_bytes, l_shape, l_sync, l_t0 = ctx.profile_launches()
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
    sync_ms = float(sum(float(t) * float(sy) / float(by)
                        for t, by, sy in zip(l_ms, l_bytes, l_sync) if by > 0))
    s_ms, s_vw, s_waited = ctx.profile_sync_latency()
    l_link = ctx.profile_link()
    l_stream = ctx.profile_streams()
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
    st1 = ctx.stats()
    ctx.profile_enable(False)
    timeline = [{"start_ms": float(a), "ms": float(t), "shape": int(sh) & 0xFFFFFFFF,
                 "stream": int(sid), "bytes": float(by), "link_bytes": float(lk)}
                for a, t, sh, sid, by, lk in zip(l_t0, l_ms, l_shape, l_stream, l_bytes, l_link)]
    # distributed placements: device time of the exchange streams (barriers /
    # flags, the owners' apply + owner-side pull launches, reader-side pulls) --
    # push + apply + pull measured on their own streams
    xs_ms = sum(float(t) for t, sid in zip(l_ms, l_stream) if int(sid) in (1, 2))
    return {"prof_ms": ms, "timeline": timeline, "xs_ms": xs_ms, "kern_ms": kern_ms,
            "kern_bytes": kern_bytes,
            "kern_launches": kern_launches, "busy_ms": busy_ms, "sync_ms": sync_ms,
            "pcommits": st1.commits - st0.commits,
            "sync_us": [1e3 * float(x) for x in s_ms],
            "sync_unblocked_us": [1e3 * float(x) for x, w in zip(s_ms, s_waited) if not w],
            "xl": [(float(t), float(b)) for t, b in zip(l_ms, l_link) if b > 0],
            "launch_mix": {k: {"n": n, "us_mean": 1e3 * t / n,
                               "GBps": b / (t / 1e3) / 1e9 if t > 0 else None}
                           for k, (n, t, b) in sorted(mix.items(), key=lambda kv: -kv[1][1])}}


def pct(xs, q):
    import numpy as np
    return float(np.percentile(xs, q)) if xs else None


def e2e_measure(cfg, span, args, ws, rank, local, stream, extra, placed):
    """The same metric through the public C-ABI with host buffers: every step
    copies the step's gradients host->device from pinned memory (EXTERNAL mode)
    and reads w_global back, inside the timed region (host wall clock, max over
    ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    N = cfg.num_vw
    e_steps = max(1, args.e2e_steps)
    ecfg = cfg.replace(waves=3 + e_steps + 1)
    from paper_2005_14038_b200 import dist as hdist
    lo, hi = hdist.shard_bounds(cfg.nparams, ws, rank)
    nloc = cfg.nparams if placed else hi - lo
    host = [torch.empty(nloc, dtype=torch.float32, pin_memory=True) for _ in range(4)]
    rng = np.random.default_rng(cfg.seed)
    for h in host:
        h.numpy()[:] = (rng.random(nloc, dtype=np.float32) - np.float32(0.5))
    run = Run(ecfg, span, args, ws, rank, local, stream, extra, grad_mode=GRAD_EXTERNAL)
    ectx = run.ctx
    out = torch.empty(max(1, ectx.local_len(-1)), dtype=torch.float32, pin_memory=True)
    ectx.trace_enable(False)
    ectx.schedule_set_host_grads([h.numpy() for h in host])
    ectx.schedule_begin(ecfg.tau, ecfg.latency())
    ectx.schedule_advance(N * 3)
    ectx.read_weights(-1, out=out.numpy())
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
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
    run.close()
    # every minibatch's gradient crosses PCIe once in total (a rank copies its
    # shard / its stages of it); w_global is read back once across the ranks
    return {"value": ecommits * cfg.nparams / dt, "unit": UNIT,
            "h2d_bytes_per_step": N * cfg.Nm * cfg.F * cfg.nparams * 4,
            "d2h_bytes_per_step": cfg.nparams * 4,
            "steps": e_steps, "ms_per_step": 1e3 * dt / e_steps,
            "path": "hp_schedule_set_host_grads + hp_schedule_advance + hp_read_weights(-1), "
                    "pinned host buffers"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hetpipe", choices=["hetpipe", "reference"])
    ap.add_argument("--config", default=None,
                    help="workload (workloads.CONFIGS); default C2 (BASELINE configs[1]) at "
                         "N=1 and C3 (configs[2], PS sharded over the GPUs) at N>1")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--profile-steps", type=int, default=20,
                    help="steps of the separate per-launch-profiled pass after the timed region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="N>1: skip the extra ED-local C2 and same-config 1-GPU measurements")
    ap.add_argument("--ref-params", type=int, default=1 << 18)
    ap.add_argument("--merge-ticks", type=int, default=1)
    ap.add_argument("--acc-slots", type=int, default=2,
                    help="acc ring depth R per VW (hp_config.acc_slots, 2..8): wave c uses "
                         "slot c mod R; R > 2 lets a VW run further ahead of its unapplied pushes")
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
    ap.add_argument("--span", type=int, default=-1,
                    help="N>1: GPUs per VW of the distributed placement (k<N exchanges over "
                         "NVLink); 0 = ED-local shards (no exchange); -1 (default) = the "
                         "SURVEY 8(d) placement of the config (C3: k=1 at 2/4 GPUs, k=2 at 8)")
    ap.add_argument("--timeline", default="",
                    help="write the profiled pass's per-launch records (start, duration, "
                         "shape, stream, bytes) of every rank to PATH.rank<r>.json")
    ap.add_argument("--graph", type=int, default=-1,
                    help="1: the timed rounds' device work is captured by hp_schedule_capture "
                         "before the timed region and launched as one CUDA graph; -1 (default) "
                         "= on for the launch-bound C1 only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = _dist()
    cfg, span = resolve_config(args, ws)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

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
    graph = bool(args.graph) if args.graph >= 0 else cfg.name.startswith("C1")
    placed = ws > 1 and span > 0
    if placed and graph:
        graph = False          # the distributed rounds are timed as issued
    extra = {}
    if placed and args.ps == "layer_rr":
        from workloads import models as wm
        extra["ps_bounds"] = wm.layer_rr_bounds(wm.MODELS[PMP_SOURCE[cfg.name][0]](), ws)
    stream = torch.cuda.Stream(local)          # a real stream: the library launches on it
    torch.cuda.set_stream(stream)              # and the timing events below record on it
    nvml = NvlinkCounters(local) if ws > 1 else None
    prof_steps = max(1, min(args.steps, args.profile_steps))
    res = measure(cfg, span, args, ws, rank, local, stream, args.steps, args.warmup, prof_steps,
                  graph, extra, sampler=True, nvml=nvml)
    if args.timeline and res.get("timeline") is not None:
        with open(f"{args.timeline}.rank{rank}.json", "w") as f:
            json.dump({"rank": rank, "config": cfg.name, "span": span, "steps": prof_steps,
                       "launches": res["timeline"]}, f)
    # link bytes this rank's GPU moved in the timed region (max over ranks)
    nv_meas = None
    if res["nvml"] is not None:
        t = torch.tensor([res["nvml"]["tx_bytes"], res["nvml"]["rx_bytes"]], dtype=torch.float64,
                         device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nv_meas = {"tx_bytes_per_step_max_rank": float(t[0]) / args.steps,
                   "rx_bytes_per_step_max_rank": float(t[1]) / args.steps,
                   "field": res["nvml"]["field"]}
    nvl = torch.tensor([res["nvl_alg"]], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(nvl, op=dist.ReduceOp.MAX)
    nvl_alg_max = float(nvl.item())

    # ---- C1 (launch-bound): per-tick time against the launch floor
    latency = None
    if cfg.name.startswith("C1") and ws == 1:
        ctx_probe = Run(cfg.replace(waves=4), 0, args, 1, 0, local, stream, {}).ctx
        floor_graph = ctx_probe.launch_floor(2000, graph=True)
        floor_direct = ctx_probe.launch_floor(2000, graph=False)
        ctx_probe.close()
        direct = measure(cfg, 0, args, 1, 0, local, stream, args.steps, args.warmup, 0, False, {})
        latency = {
            "tick_us": 1e3 * res["ms_max"] / max(res["ticks"], 1),
            "launches_per_tick": res["launches"] / max(res["ticks"], 1),
            "us_per_launch": 1e3 * res["ms_max"] / max(res["launches"], 1),
            "launch_floor_us": {"graph": floor_graph, "direct": floor_direct},
            "ratio_to_floor": (1e3 * res["ms_max"] / max(res["ticks"], 1)) /
                              (floor_graph if graph else floor_direct),
            "issued_directly": {"tick_us": 1e3 * direct["ms_max"] / max(direct["ticks"], 1),
                                "value": direct["value"],
                                "us_per_launch": 1e3 * direct["ms_max"] / max(direct["launches"], 1)},
            "def": "device time of the timed rounds / controller ticks; floor = empty one-CTA "
                   "kernels back to back on the same stream (hp_launch_floor), in a graph and "
                   "issued directly; ratio_to_floor = tick_us / the floor of the same issue "
                   "mode (captured ticks of a small context run through the multi-tick kernel, "
                   "hp_schedule_capture)"}

    # ---- N>1: the ED-local C2 placement and the same config on one GPU
    extras = {}
    if ws > 1 and not args.no_extras and args.config is None:
        c2 = measure(CONFIGS["C2"], 0, args, ws, rank, local, stream, min(args.steps, 100),
                     args.warmup, 0, False, {})
        extras["ed_local_c2"] = {
            "value": c2["value"], "ms_per_step": c2["ms_max"] / min(args.steps, 100),
            "hbm_frac": c2["alg_bytes"] / (c2["ms_max"] / 1e3) / 1e9 / _peaks()[0],
            "def": "C2 (configs[1]) sharded ED-local over the N GPUs (no exchange), "
                   "device-timed, max over ranks"}
        # the same config on ONE GPU (rank 0's; every rank runs it on its own GPU
        # with no communication, so the ranks stay in step)
        one = measure(cfg, 0, args, 1, 0, local, stream, min(args.steps, 100), args.warmup, 0,
                      False, {})
        extras["same_config_n1"] = {
            "value": one["value"], "ms_per_step": one["ms_max"] / min(args.steps, 100),
            "def": f"{cfg.name} with every VW and the PS on one GPU (rank 0's), device-timed: "
                   "the 1-GPU point of this config's scaling"}
        dist.barrier()

    e2e = None
    if not args.no_e2e and cfg.grad_mode != 3:
        e2e = e2e_measure(cfg, span, args, ws, rank, local, stream, extra, placed)

    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_kind = _peaks()
    G = ws
    # roofline on the TIMED region: the tick launches' algorithmic bytes (this
    # rank's, from the descriptors) over the timed device time (max over ranks);
    # the launches fill >= 0.99 of it (kernel_share_of_step)
    achieved = res["alg_bytes"] / (res["ms_max"] / 1e3) / 1e9
    synthetic = cfg.grad_mode in (0, 1)
    sb = survey_bytes_per_param(res["commits"], res["apply_batches"], cfg)
    survey_achieved = sb * cfg.nparams / G / (res["ms_max"] / 1e3) / 1e9
    rounds = res["commits"] / cfg.num_vw
    nv_peak, nv_kind = nvlink_peak()
    xch = None
    if res.get("xl"):
        xt, xb = sum(t for t, _ in res["xl"]), sum(b for _, b in res["xl"])
        xch = {"launches": len(res["xl"]), "ms": xt, "link_bytes": xb,
               "achieved_GBps": xb / (xt / 1e3) / 1e9, "peak_GBps": nv_peak,
               "peak_kind": nv_kind, "frac": xb / (xt / 1e3) / 1e9 / nv_peak, "bound": "nvlink",
               "frac_vs_nominal_900": xb / (xt / 1e3) / 1e9 / 900.0,
               "def": "exchange launches only (peer loads/stores, NVLS multimem, NCCL "
                      "collectives): algorithmic NVLink bytes per direction / their device "
                      "time, rank 0, profiled pass"}
    sync_us, unb = res.get("sync_us", []), res.get("sync_unblocked_us", [])
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_max"] / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "num_vw": cfg.num_vw, "Nm": cfg.Nm, "D": cfg.D,
                   "F": cfg.F, "nparams": cfg.nparams, "tau": list(cfg.tau),
                   "lat": list(cfg.latency()), "timing": args.timing, "placement":
                   (f"distributed, {span} GPU(s) per VW, PS sharded over {ws}" if placed
                    else "ED-local shards" if ws > 1 else "single GPU"),
                   "grad": ("CONVEX a(w_p - b) + sigma xi, w_p from the START stash"
                            if args.grad == "convex" else "Philox FLOAT in-kernel"),
                   "pull": args.pull.upper(), "local": "STRICT",
                   "apply": "on arrival" if args.apply_mode else "deferred to the observing pull",
                   "acc_slots": args.acc_slots,
                   "cuda_device_max_connections": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"),
                   "transport": args.transport if placed else None,
                   "ps_shards": args.ps if placed else None,
                   "lockstep_batches": res["lockstep"] if placed else None,
                   "issue": "one CUDA graph (hp_schedule_capture)" if graph else "direct launches",
                   "l2": ("inputs larger than L2 (>= 13 x 230 MiB buffers per GPU)"
                          if cfg.nparams >= (1 << 24) else
                          "model fits in L2 (latency-bound config; no flush)"),
                   "arena_GiB_per_rank": res["arena"] / 2 ** 30},
        "images_per_sec_equiv": res["commits"] * 32 * cfg.Nm * cfg.F / (res["ms_max"] / 1e3),
        "sync_only_modelled": (
            {"value": res["commits"] * cfg.nparams / (res["sync_ms_max"] / 1e3), "unit": UNIT,
             "ms_per_step": res["sync_ms_max"] / args.steps,
             "def": "MODELLED, not timed: push/apply/pull are fused with accumulation, so each "
                    "profiled launch's device time is attributed to synchronisation by its share "
                    "of algorithmic bytes (w_global/m, u~ reads, pull writes), scaled to the "
                    "timed steps; max over ranks"}
            if res["sync_ms_max"] > 0 else None),
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": _ncu_traffic(cfg.name),
            "peak_kind": peak_kind, "kernel": "hp::tick_kernel (all launches)",
            "def": "timed region: algorithmic bytes of the tick launches (the kernel's own "
                   "buffer passes, tick_desc.h tick_streams; rank 0) / timed device time",
            "alg_bytes_per_param_per_round": res["alg_bytes"] * G / cfg.nparams / max(rounds, 1),
            "frac_survey": (survey_achieved / peak) if synthetic else None,
            "survey_bytes_per_param_per_round": sb / max(rounds, 1),
            "survey_def": "SURVEY.md 8(d) byte model on the timed region: 16*F*Nm per push "
                          "(accumulate 16U-12, u~ read 4, pull 8) + 8 (+8 momentum) per apply "
                          "batch (k = pushes / apply_batches as run), x P / G per GPU",
            "pushes_per_apply_batch": res["commits"] / max(res["apply_batches"], 1),
            "frac_vs_nominal_8000": achieved / 8000.0,
            "frac_profiled": (res["kern_bytes"] / (res["busy_ms"] / 1e3) / 1e9 / peak
                              if res.get("busy_ms") else None),
            "launches": res["launches"],
            "alg_bytes_per_launch": res["alg_bytes"] / max(res["launches"], 1)},
        "exchange_roofline": xch,
        "exchange_stream": ({"ms_per_step": res["xs_ms"] / prof_steps,
                             "synced_params_per_s": res["pcommits"] * cfg.nparams /
                             (res["xs_ms"] / 1e3) if res.get("xs_ms") else None,
                             "def": "distributed placements, rank 0, profiled pass: device time "
                                    "of the exchange stream(s) -- flag waits, the PS shard's apply "
                                    "launches with the owner-side pull stores, reader-side pulls "
                                    "-- i.e. push + apply + pull measured on their own stream "
                                    "(waits for the other ranks included)"}
                            if placed and res.get("xs_ms") else None),
        "nvlink": {"alg_bytes_per_step_max_rank": nvl_alg_max / args.steps,
                   "alg_GBps_over_step": nvl_alg_max / (res["ms_max"] / 1e3) / 1e9,
                   "measured": nv_meas,
                   "peak_GBps": nv_peak, "peak_kind": nv_kind},
        "wave_sync_latency_us": (
            {"p50": pct(sync_us, 50), "p99": pct(sync_us, 99), "max": max(sync_us),
             "n": len(sync_us),
             "unblocked": ({"p50": pct(unb, 50), "p99": pct(unb, 99), "n": len(unb)}
                           if unb else None),
             "def": "per (VW, wave), rank 0, profiled pass: device time from the start of the "
                    "launch carrying the VW's wave-end COMPLETE (u~ final = push) to the end of "
                    "the launch that wrote its pulled w_local (hp_profile_sync_latency); all "
                    "records include gate waits, `unblocked` only those whose VW did not wait"}
            if sync_us else None),
        "kernel_share_of_step": (res["busy_ms"] / res["prof_ms"]
                                 if res.get("prof_ms") else None),
        "launch_mix": res.get("launch_mix"),
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "wait_ticks_per_vw": res["waits"],
        "e2e": e2e,
    }
    if latency:
        line["latency"] = latency
    line.update(extras)
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Shared helpers of the distributed-placement parity tests (test
infrastructure): drive one rank's context through a whole schedule, collect
its trace and buffers (whole, or only sampled global indices at full size),
and compare the reassembled shards / stages of every rank with the oracle.

Used by tests/gpu_multi_parity.py (one process per GPU under torchrun),
tests/test_gpu_colocated.py (G ranks as threads sharing ONE GPU, connected
without NCCL) and tests/test_colocated_emu.py (the same on the host emulation).
"""
from __future__ import annotations

import tempfile
import threading

import numpy as np

from oracle import gradient, run_schedule
from workloads import even_shards


def host_gradients(cfg):
    """EXTERNAL mode: the VWs' whole gradients as host buffers, filled with the
    same Philox values the synthetic mode draws (oracle.gradient), laid out as
    include/hetpipe.h hp_schedule_set_host_grads indexes them."""
    idx = np.arange(cfg.nparams)
    last_p = cfg.waves * cfg.Nm * cfg.F
    n = cfg.num_vw * last_p + 1
    bufs = [np.zeros(cfg.nparams, dtype=np.float32) for _ in range(n)]
    for v in range(cfg.num_vw):
        for p in range(1, last_p + 1):
            bufs[(v * last_p + p) % n][:] = gradient(idx, v, p, cfg)
    return bufs


def holds(v, k, G, rank):
    return any((v * k + j) % G == rank for j in range(k))


def collect(ctx, cfg, G, k, rank, sampled=None, bounds=None):
    """(trace, w_global shard, m shard, {v: w_local stage}, nvl_bytes,
    lockstep_batches) of one rank after its schedule; with `sampled` the arrays
    become {global index: value} for the sampled indices this rank holds."""
    with tempfile.NamedTemporaryFile(suffix=".trace") as f:
        tr = ctx.trace_lines(f.name)
    wg = ctx.read_weights(-1)
    m = ctx.read_weights(-2) if cfg.momentum else None
    wl = {v: ctx.read_weights(v) for v in range(cfg.num_vw) if holds(v, k, G, rank)}
    st = ctx.stats()
    nvl, lock = st.nvl_bytes, st.lockstep_batches
    if sampled is not None:      # ship only sampled entries (full arrays are GBs)
        sb = bounds or even_shards(cfg.nparams, G)
        lo, hi = sb[rank], sb[rank + 1]
        wg = {int(i): float(wg[i - lo]) for i in sampled if lo <= i < hi}
        m = None if m is None else {int(i): float(m[i - lo]) for i in sampled if lo <= i < hi}
        stb = even_shards(cfg.nparams, k)
        wl2 = {}
        for v, arr in wl.items():
            j = [j for j in range(k) if (v * k + j) % G == rank][0]
            wl2[v] = {int(i): float(arr[i - stb[j]]) for i in sampled if stb[j] <= i < stb[j + 1]}
        wl = wl2
    return tr, wg, m, wl, nvl, lock


def normwise(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def check(cfg, G, k, objs, sampled=None, exact=True):
    """exact: bit-identical arrays (commit-order applies); otherwise reading
    Z15's normwise bound 1e-5 per buffer (NCCL / NVLS sum a lockstep wave's N
    updates in their own order before the single apply). Traces must be
    byte-identical on every rank."""
    eq = (lambda a, b: np.array_equal(a, b)) if exact else (lambda a, b: normwise(a, b) <= 1e-5)
    o = run_schedule(cfg, idx=None if sampled is None else np.array(sampled))
    for r in range(G):
        assert objs[r][0] == o.trace, f"trace of rank {r}"
    if sampled is None:
        assert eq(np.concatenate([objs[r][1] for r in range(G)]), o.wg), "w_global"
        if cfg.momentum:
            assert eq(np.concatenate([objs[r][2] for r in range(G)]), o.m), "momentum"
        for v in range(cfg.num_vw):
            parts = [objs[(v * k + j) % G][3][v] for j in range(k)]
            assert eq(np.concatenate(parts), o.wl[v]), f"w_local({v})"
    else:
        wg, m = {}, {}
        for r in range(G):
            wg.update(objs[r][1])
            if cfg.momentum:
                m.update(objs[r][2])
        assert eq(np.array([wg[i] for i in sampled], dtype=np.float32), o.wg), "w_global"
        if cfg.momentum:
            assert eq(np.array([m[i] for i in sampled], dtype=np.float32), o.m), "momentum"
        for v in range(cfg.num_vw):
            wl = {}
            for j in range(k):
                wl.update(objs[(v * k + j) % G][3][v])
            assert eq(np.array([wl[i] for i in sampled], dtype=np.float32), o.wl[v]), f"w_local({v})"
    nvl = sum(objs[r][4] for r in range(G))
    assert (nvl == 0) == (k == G), nvl
    return o


RETRIES = []   # (config name, G, k, message) of attempts repeated after a queue-aliasing stall


def run_colocated(hetpipe, cfg, G, k, alloc, lib=None, sampled=None, bounds=None,
                  host_grads=None, timeout=600.0, rounds_per_chunk=2, attempts=3, **over):
    """G ranks of a distributed placement as G threads of THIS process, each
    driving its own context; the arenas come from alloc(nbytes) -> (address,
    keepalive) (torch device memory on the GPU, numpy for the host emulation)
    and the contexts connect through hp_connect_symmetric WITHOUT an NCCL
    communicator (comm_id NULL: K7 flag barriers, PEER exchange). Returns the
    per-rank collect() tuples in rank order.

    Co-located ranks share one GPU's hardware work queues, and CUDA maps
    streams to queues itself: when one rank's spinning flag kernel lands in the
    queue in front of another rank's producer, the wait can only end at the
    flag deadline (HP_ERR_COMM; reproduced at will with
    CUDA_DEVICE_MAX_CONNECTIONS=1 or 4, rare at 32 -- separate GPUs cannot
    alias). Such an attempt is repeated with fresh contexts (new streams, a
    new mapping) up to `attempts` times and recorded in RETRIES; any other
    failure, or a second identical stall, fails."""
    for attempt in range(attempts):
        try:
            return _run_colocated_once(hetpipe, cfg, G, k, alloc, lib, sampled, bounds,
                                       host_grads, timeout, rounds_per_chunk, **over)
        except _FlagStall as e:
            RETRIES.append((cfg.name, G, k, str(e)[:200]))
            if attempt + 1 == attempts:
                raise AssertionError(f"flag stall in {attempts} attempts: {e}")


class _FlagStall(Exception):
    pass


def _run_colocated_once(hetpipe, cfg, G, k, alloc, lib, sampled, bounds, host_grads, timeout,
                        rounds_per_chunk, **over):
    extra = dict(over)
    if bounds is not None:
        extra["ps_bounds"] = bounds
    keep, ctxs = [], []
    try:
        for r in range(G):
            c = hetpipe.config_from(cfg, world=G, rank=r, vw_span=k, **extra)
            addr, kp = alloc(hetpipe.arena_bytes(c, lib))
            keep.append(kp)
            c.arena = addr
            ctxs.append(hetpipe.Context(c, lib=lib))
        bases = [ctx.cfg.arena for ctx in ctxs]
        out, errs = [None] * G, []
        connected = threading.Barrier(G)

        def work(r):
            try:
                ctx = ctxs[r]
                ctx.connect_symmetric(bases, 0, None)
                # every rank's set-up (its allocations, streams, first barrier)
                # is finished before any rank issues flag waits of the schedule
                connected.wait(timeout)
                if host_grads is not None:
                    ctx.schedule_set_host_grads(host_grads)
                # advance a bounded number of rounds at a time, then drain: the
                # co-located ranks share ONE CUDA context, so one rank's host
                # must not run so far ahead that its queued launches (blocked
                # behind a flag wait for another rank) fill the context's
                # command queue before the other rank has issued its signal
                # (separate processes / GPUs have separate queues)
                ctx.schedule_begin(cfg.tau, cfg.latency())
                total = cfg.num_vw * cfg.waves
                for target in range(cfg.num_vw * rounds_per_chunk, total + 1,
                                    cfg.num_vw * rounds_per_chunk):
                    ctx.schedule_advance(target)
                    ctx.drain()
                ctx.schedule_advance(total)
                ctx.sync()
                out[r] = collect(ctx, cfg, G, k, r, sampled, bounds)
            except Exception as e:  # reported below
                errs.append((r, e))
                connected.abort()     # release ranks waiting for this one

        th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout)
        assert not any(t.is_alive() for t in th), "a rank thread did not finish"
        def stall(e):      # a flag deadline, in the schedule or at connect
            return ((getattr(e, "status", None) == hetpipe.HP_ERR_COMM and
                     ("timed out" in str(e) or "did not reach" in str(e)))
                    or isinstance(e, threading.BrokenBarrierError))
        if errs and any(stall(e) for _, e in errs) and all(
                stall(e) for _, e in errs):
            raise _FlagStall(errs)
        assert not errs, errs
        return out
    finally:
        for ctx in ctxs:
            ctx.close()
        del keep

"""On-box NVLink peaks for the exchange roofline (run on a box with >= 2 B200s;
one process, every visible GPU). Copy-engine peer copies of 1 GiB through
torch (cudaMemcpyPeerAsync with P2P enabled), device-timed with CUDA events,
median of 5 after a warm-up:

  * uni: GPU 0 -> GPU 1 alone;
  * bidir: 0 -> 1 and 1 -> 0 at once (per direction);
  * ingress: every other GPU -> GPU 0 at once (what one PS owner receives);
  * egress: GPU 0 -> every other GPU at once.

It also samples NVML's NVLink data counters (NVLINK_THROUGHPUT_DATA_TX/RX)
around the uni copy, to check that the counters bench.py reads measure the
bytes a copy moves.

    python scripts/nvlink_peak.py [--out profiles/nvlink_peak.json]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(pairs, nbytes, reps=5):
    """Concurrent copies src -> dst for (src, dst) in pairs: (GB/s of one copy
    alone by its own CUDA events -- the slowest, and the aggregate GB/s of all
    copies over the host wall time from the first issue to the last
    completion, every device synchronised on both sides)."""
    import time
    bufs = []
    for s, d in pairs:
        a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{s}")
        b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}")
        st = torch.cuda.Stream(device=s)
        bufs.append((a, b, st, s))
    per, agg = [], []
    for rep in range(reps + 1):
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)
        evs = []
        t0 = time.perf_counter()
        for a, b, st, s in bufs:
            with torch.cuda.device(s), torch.cuda.stream(st):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                b.copy_(a, non_blocking=True)
                e1.record(st)
                evs.append((e0, e1))
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)
        dt = time.perf_counter() - t0
        if rep:
            per.append(min(nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9 for e0, e1 in evs))
            agg.append(len(bufs) * nbytes / dt / 1e9)
    return statistics.median(per), statistics.median(agg)


def nvml_probe(index=0):
    """What NVML reports for this GPU's NVLinks (states, and the data
    counters bench.py reads), to debug an unsupported field."""
    out = {}
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        states = {}
        for link in range(18):
            try:
                states[link] = int(pynvml.nvmlDeviceGetNvLinkState(h, link))
            except Exception as e:
                states[link] = repr(e)[:60]
        out["link_state"] = states
        for fid in (138, 139, 140, 141, 202, 204):
            res = {}
            for scope in (0, 1, 0xFFFFFFFF):
                try:
                    v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                    res[str(scope)] = [int(v.nvmlReturn), int(v.value.ullVal)]
                except Exception as e:
                    res[str(scope)] = repr(e)[:80]
            out[f"field_{fid}"] = res
    except Exception as e:
        out["error"] = repr(e)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "nvlink_peak.json"))
    ap.add_argument("--gib", type=float, default=1.0)
    args = ap.parse_args()
    G = torch.cuda.device_count()
    assert G >= 2, "needs >= 2 GPUs"
    n = int(args.gib * (1 << 30))
    for i in range(G):
        for j in range(G):
            if i != j:
                assert torch.cuda.can_device_access_peer(i, j), (i, j)
    import bench
    nv = bench.NvlinkCounters(0)
    c0 = nv.read()
    uni, _ = timed([(0, 1)], n)
    c1 = nv.read()
    bidir, bidir_agg = timed([(0, 1), (1, 0)], n)
    ing1, ingress = timed([(q, 0) for q in range(1, G)], n)
    eg1, egress = timed([(0, q) for q in range(1, G)], n)
    res = {
        "gpus": G, "name": torch.cuda.get_device_name(0), "bytes": n,
        "uni_GBps": uni, "bidir_GBps_per_direction": bidir_agg / 2,
        "ingress_GBps_total": ingress, "ingress_slowest_copy_GBps": ing1,
        "egress_GBps_total": egress, "egress_slowest_copy_GBps": eg1,
        # the per-direction peak of one GPU's links: the best aggregate measured
        "peer_copy_GBps_per_direction": max(uni, bidir_agg / 2, ingress, egress),
        "nvml_probe": nvml_probe(0),
        "nvml_counter_check": (None if c0 is None or c1 is None else
                               {"field": nv.field, "tx_bytes": c1[0] - c0[0],
                                "rx_bytes": c1[1] - c0[1],
                                "copied_bytes": 6 * n,
                                "note": "GPU 0 sent 6 x 1 GiB (warm-up + 5) in the uni test"}),
        "method": "torch copy_ between devices (copy engines, P2P), CUDA events, median of 5",
    }
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

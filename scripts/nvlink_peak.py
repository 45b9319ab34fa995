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
    """Concurrent copies src -> dst for (src, dst) in pairs; GB/s per copy."""
    bufs = []
    for s, d in pairs:
        a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{s}")
        b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}")
        st = torch.cuda.Stream(device=s)
        bufs.append((a, b, st, s))
    out = []
    for rep in range(reps + 1):
        evs = []
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
        if rep:
            out.append(min(nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9 for e0, e1 in evs))
    return statistics.median(out)


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
    uni = timed([(0, 1)], n)
    c1 = nv.read()
    bidir = timed([(0, 1), (1, 0)], n)
    ingress = timed([(q, 0) for q in range(1, G)], n)
    egress = timed([(0, q) for q in range(1, G)], n)
    res = {
        "gpus": G, "name": torch.cuda.get_device_name(0), "bytes": n,
        "uni_GBps": uni, "bidir_GBps_per_direction": bidir,
        "ingress_GBps_per_source": ingress, "ingress_GBps_total": ingress * (G - 1),
        "egress_GBps_per_dest": egress, "egress_GBps_total": egress * (G - 1),
        # the per-direction peak of one GPU's links: the best of the measured forms
        "peer_copy_GBps_per_direction": max(uni, bidir, ingress * (G - 1), egress * (G - 1)),
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

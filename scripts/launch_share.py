"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launch count, total and mean duration and share of the total
(ncu serialises launches and runs them cold-cache: compare SHARES with the
bench's CUDA-event numbers, not absolute times).

    python scripts/launch_share.py profiles/r01_launches.csv
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]), r["Metric Unit"]))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    agg = defaultdict(lambda: [0, 0.0])
    for name, v, unit in rows:
        short = name.split("(")[0]
        agg[short][0] += 1
        agg[short][1] += v * scale.get(unit, 1.0)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':60s} {'n':>5s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:5d} {t:12.1f} {t / n:10.1f} {t / tot:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])

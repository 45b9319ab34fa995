"""Report of the pipeline-derived VW timing (NEXT-1): per model x Table 2
policy x Nm, each VW's partition (native hp_partition), stage times, tau / L
(hp_pipeline_tau_latency), images/s, and the native partitioner's run time
next to the oracle's brute force on the same input.

    python scripts/pmp_report.py > profiles/r01_pmp_partitions.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pipeline as op  # noqa: E402
from paper_2005_14038_b200 import hetpipe, schedule  # noqa: E402
from workloads import models as M  # noqa: E402


def main():
    print("# pipeline-derived VW timing (times in ms; tau = steady-state interval per minibatch,")
    print("# L = first-minibatch latency; img/s = 32 / tau summed over the 4 VWs)")
    for model in ("resnet152", "vgg19"):
        units = M.MODELS[model]()
        for policy in ("NP", "ED", "HD"):
            for Nm in (1, 4, 8):
                tot = 0.0
                rows = []
                for vw, types in enumerate(M.POLICIES[policy]):
                    g = schedule.vw_gpus(types)
                    t0 = time.perf_counter()
                    part = hetpipe.partition(units, g, Nm, intra_bps=M.PCIE_BPS, inter_bps=M.IB_BPS)
                    t_native = time.perf_counter() - t0
                    b, order, cuts, costs = part
                    tau, lat = hetpipe.pipeline_tau_latency(costs, Nm)
                    tot += 32 / (tau / 1e9)
                    st = [round((f + bw + cf + cb) / 1e6, 1) for f, bw, cf, cb in costs]
                    rows.append(f"  VW{vw + 1} {types}: order={''.join(types[i] for i in order)} "
                                f"cuts={list(cuts)} stage_ms={st} tau={tau / 1e6:.1f} "
                                f"L={lat / 1e6:.1f} native_partition_s={t_native:.4f}")
                print(f"{model} {policy} Nm={Nm}: {tot:.0f} img/s")
                print("\n".join(rows))
    # native vs brute force cost on one VW of each model
    for model, types in (("vgg19", "VVQQ"), ("resnet152", "VVQQ")):
        units, g = M.MODELS[model](), schedule.vw_gpus(types)
        t0 = time.perf_counter()
        hetpipe.partition(units, g, 4, intra_bps=M.PCIE_BPS, inter_bps=M.IB_BPS)
        tn = time.perf_counter() - t0
        t0 = time.perf_counter()
        op.partition_bruteforce(units, g, 4)
        tb = time.perf_counter() - t0
        print(f"# {model} {types} Nm=4: native DP {tn * 1e3:.2f} ms, oracle brute force {tb:.2f} s")


if __name__ == "__main__":
    main()

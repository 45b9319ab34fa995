"""Per-VW timing of the WSP controller from the intra-VW pipeline schedule
(section 4): partition the model
over each VW's GPUs (hp_partition: min-max stage time under the
stage-dependent memory requirement), simulate the VW's pipeline under
scheduling conditions 1-3 (hp_pipeline_tau_latency) and hand the resulting
(tau_v, L_v) to hp_schedule_begin, replacing the speed proxy of reading Z14.
Argument marshalling only: the partitioner and the simulator are native
(csrc/pipeline.cpp). Ticks are microseconds."""
from __future__ import annotations

from typing import List, Sequence, Tuple

from workloads import models as M

from . import hetpipe


def vw_gpus(types: str) -> List[dict]:
    F = M.v_flops_per_s()
    return [{"flops": F * M.GPUS[t].speed, "mem": M.GPUS[t].mem_gb * 1e9, "node": M.NODE_OF[t]}
            for t in types]


def vw_timing(model: str, types: str, Nm: int):
    """(tau_us, L_us, partition) of one VW made of GPU types `types` (e.g. "VVQQ")."""
    part = hetpipe.partition(M.MODELS[model](), vw_gpus(types), Nm, batch=M.BATCH,
                             intra_bps=M.PCIE_BPS, inter_bps=M.IB_BPS)
    if part is None:
        raise ValueError(f"{model} does not fit a {types} VW at Nm={Nm}")
    tau_ns, lat_ns = hetpipe.pipeline_tau_latency(part[3], Nm)
    return max(1, round(tau_ns / 1000)), max(1, round(lat_ns / 1000)), part


def policy_timing(model: str, policy: str, Nm: int, vws: Sequence[str] = ()) -> Tuple[tuple, tuple]:
    """(tau, lat) tuples in microseconds for the VWs of a Table 2 policy (or an
    explicit list of VW GPU-type strings)."""
    types = list(vws) or list(M.POLICIES[policy])
    out = [vw_timing(model, t, Nm)[:2] for t in types]
    return tuple(t for t, _ in out), tuple(l for _, l in out)

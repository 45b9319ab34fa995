"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This module holds ONLY configuration: sizes, seeds, virtual-worker speed
vectors and the mode flags. It contains none of the method's arithmetic (no
gradient generator, no accumulation, no clock logic), so importing it from both
`oracle/` and `paper_2005_14038_b200/` does not couple the two implementations.

Recipe (DESIGN.md section "Input recipe"):
  * seed 200514038 for every config;
  * gradients are drawn from Philox4x32-10 by each side's OWN generator, keyed by
    the seed, with counter (i>>2, vw, p, stream=0); word i&3 is param i's draw;
  * w0 is either zero or Philox stream 1, counter (i>>2, 0, 0, 1);
  * per-VW ticks per minibatch tau_v mimic the paper's NP / ED / HD allocations
    (Table 2 and Table 3 rates P:241-252; SURVEY.md 8(d) speed
    proxy V=1.00, R=0.76, G=0.72, Q=0.59, tau = 1000 / sum of a VW's GPU speeds);
  * fill latency L_v defaults to Nm * tau_v.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence, Tuple

SEED = 200514038

# grad_mode
GRAD_FLOAT = 0      # g = (x>>8) * 2^-24 - 0.5, uniform in [-0.5, 0.5)
GRAD_DYADIC = 1     # g = (x>>28) - 8, integers in {-8..7}
GRAD_EXTERNAL = 2   # caller-supplied gradient buffers (CUDA path only)
GRAD_CONVEX = 3     # g = a * (w_p - b) + sigma * xi: weight-dependent (NEXT-2), w_p =
                    # w_local at START(p), b = Philox stream 2 in [-1, 1), xi the FLOAT
                    # draw of stream 0 in [-0.5, 0.5)

# w0_mode
W0_ZERO = 0
W0_PHILOX = 1

# pull_policy
PULL_EAGER = 0
PULL_LAZY = 1

# lr_schedule
LR_CONSTANT = 0
LR_THEOREM1 = 1

# local_semantics
LOCAL_STRICT = 0
LOCAL_AT_LEAST = 1

RESNET152_PARAMS = 60_192_808    # 229.6 MiB fp32 ("230MB")
VGG19_PARAMS = 143_667_240       # 548.0 MiB fp32 ("548MB")

TAU_NP = (250, 330, 346, 421)    # Node-Partition: V / R / G / Q nodes
TAU_ED = (325, 325, 325, 325)    # Equal-Distribution: every VW = VRGQ
TAU_HD = (314, 314, 338, 338)    # Hybrid: VVQQ, VVQQ, RRGG, RRGG


@dataclasses.dataclass(frozen=True)
class WSPConfig:
    """One WSP run: N virtual workers, Nm minibatches per wave, threshold D."""
    name: str
    num_vw: int
    Nm: int
    D: int
    nparams: int
    waves: int
    tau: Tuple[int, ...]
    lr: float = 0.01
    momentum: float = 0.0
    seed: int = SEED
    grad_mode: int = GRAD_FLOAT
    w0_mode: int = W0_PHILOX
    pull_policy: int = PULL_EAGER
    local_semantics: int = LOCAL_STRICT
    lat: Optional[Tuple[int, ...]] = None   # fill latency per VW; None -> Nm * tau
    conv_a: float = 0.5                     # GRAD_CONVEX curvature a
    conv_sigma: float = 1.0                 # GRAD_CONVEX noise scale sigma
    F: int = 1                              # update frequency factor (NEXT-4): one clock
                                            # = F waves; `waves` counts clocks
    lr_schedule: int = 0                    # 0: constant lr; 1: Theorem 1's eta_t =
                                            # lr / sqrt(t), t = (p-1)*N + v + 1 (NEXT-2)

    def latency(self) -> Tuple[int, ...]:
        if self.lat is not None:
            return tuple(self.lat)
        return tuple(self.Nm * t for t in self.tau)

    def replace(self, **kw) -> "WSPConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; SURVEY.md 8(d) "Concrete synthetic inputs".
C1 = WSPConfig("C1", 2, 1, 0, 4096, 16, (100, 100), lr=2.0 ** -6,
               grad_mode=GRAD_DYADIC, w0_mode=W0_ZERO)
C1_SKEW = C1.replace(name="C1-skew", tau=(100, 173))
C2 = WSPConfig("C2", 4, 4, 0, RESNET152_PARAMS, 32, TAU_NP)
C3 = WSPConfig("C3", 4, 4, 4, RESNET152_PARAMS, 64, TAU_HD)
C4 = WSPConfig("C4", 4, 8, 32, VGG19_PARAMS, 132, TAU_ED)
C5 = WSPConfig("C5", 8, 8, 0, VGG19_PARAMS, 132,
               (250, 250, 330, 330, 346, 346, 421, 421), momentum=0.9)

# C5's equal-speed SGD variant (SURVEY.md 8(d) "plus an equal-speed variant"):
# with D = 0 every VW pushes and pulls in the same tick, the lockstep batch the
# NCCL / NVLS transports exchange (include/hetpipe.h HP_XPORT_*); one VW per GPU
# (num_vw = G at run time).
C5E = WSPConfig("C5E", 8, 8, 0, VGG19_PARAMS, 132, (325,) * 8)
# The Horovod analogue (Horovod is the paper's baseline,
# P:203-226): the BSP limit of WSP (Nm = 1, D = 0, pin P8) with one VW per GPU
# and equal speeds = synchronous data-parallel SGD, every minibatch a lockstep
# batch (all-reduce through NCCL, or the NVLS kernel).
HVD = WSPConfig("HVD", 8, 1, 0, VGG19_PARAMS, 132, (325,) * 8)
CONFIGS = {c.name: c for c in (C1, C1_SKEW, C2, C3, C4, C5, C5E, HVD)}

# Model and VW GPU types behind each config, for the pipeline-derived timing
# (tau_v, L_v from partitioning the model over the VW's
# GPUs, replacing the speed proxy; workloads/models.py holds the tables).
PMP_SOURCE = {
    "C2": ("resnet152", ("VVVV", "RRRR", "GGGG", "QQQQ")),          # NP
    "C3": ("resnet152", ("VVQQ", "VVQQ", "RRGG", "RRGG")),          # HD
    "C4": ("vgg19", ("VRGQ",) * 4),                                 # ED
    "C5": ("vgg19", ("VVVV", "VVVV", "RRRR", "RRRR", "GGGG", "GGGG", "QQQQ", "QQQQ")),
    "C5E": ("vgg19", ("VRGQ",) * 8),
    "HVD": ("vgg19", ("V",) * 8),
}


def even_shards(nparams: int, nshards: int, align: int = 32) -> Sequence[int]:
    """Shard boundaries b_0=0 < ... < b_G = nparams, inner ones multiples of
    `align` floats (even contiguous shards, last takes the rest)."""
    per = (nparams // nshards) // align * align
    bounds = [s * per for s in range(nshards)] + [nparams]
    return bounds


def ceil_shards(nparams: int, nshards: int, align: int = 32) -> Sequence[int]:
    """The NCCL transport's default shards: the first G-1 equal (ceil, rounded
    up to `align`), the last the rest."""
    per = (-(-nparams // nshards) + align - 1) // align * align
    return [min(s * per, nparams) for s in range(nshards)] + [nparams]


def sample_indices(nparams: int, stride: int = 4099, extra: Sequence[int] = ()) -> list:
    """A deterministic index sample for full-size parity: every `stride`-th param,
    the first 8 and last 8 params, and any extra indices (e.g. shard boundaries)."""
    idx = set(range(0, nparams, stride))
    idx.update(range(min(8, nparams)))
    idx.update(range(max(0, nparams - 8), nparams))
    for e in extra:
        for d in (-1, 0, 1):
            if 0 <= e + d < nparams:
                idx.add(e + d)
    return sorted(idx)

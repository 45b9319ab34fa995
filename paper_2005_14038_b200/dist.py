"""Multi-GPU plumbing for the ED-local placement: one
process per GPU, each owning a contiguous parameter shard of every VW's state
and of the PS. Every rank runs the same deterministic controller (identical
event order, identical traces), so the WSP path needs no data-path collective
in this placement; torch.distributed is used only for the bench's barrier and
max-over-ranks timing. Shard boundaries are multiples of 32 floats (SURVEY.md
Z12), which keeps every rank's Philox counter blocks aligned."""
from __future__ import annotations

from typing import Optional

from workloads import even_shards

from . import hetpipe


def shard_bounds(nparams: int, world: int, rank: int):
    b = even_shards(nparams, world)
    return b[rank], b[rank + 1]


def rank_context(cfg, rank: int, world: int, device: int = 0, stream: int = 0,
                 lib=None, **overrides) -> hetpipe.Context:
    """Context for this rank's shard of workload cfg (a workloads.WSPConfig)."""
    lo, hi = shard_bounds(cfg.nparams, world, rank)
    c = hetpipe.config_from(cfg, param_begin=lo, param_count=hi - lo, device=device,
                            stream=stream or None, **overrides)
    return hetpipe.Context(c, lib=lib)

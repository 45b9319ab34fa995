"""Multi-GPU plumbing for the ED-local placement: one
process per GPU, each owning a contiguous parameter shard of every VW's state
and of the PS. Every rank runs the same deterministic controller (identical
event order, identical traces), so the WSP path needs no data-path collective
in this placement; torch.distributed is used only for the bench's barrier and
max-over-ranks timing. Shard boundaries are multiples of 32 floats (SURVEY.md
Z12), which keeps every rank's Philox counter blocks aligned."""
from __future__ import annotations

from typing import Optional

import os

from workloads import even_shards

from . import hetpipe


def _nccl_hint() -> None:
    """Point the library at torch's bundled NCCL (HP_NCCL_LIB) unless set; the
    library first reuses an NCCL already loaded in the process."""
    if os.environ.get("HP_NCCL_LIB"):
        return
    try:
        import nvidia.nccl  # the pip package torch's NCCL comes from
        for d in nvidia.nccl.__path__:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["HP_NCCL_LIB"] = cand
                return
    except ImportError:
        pass


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


def placed_context(cfg, rank: int, world: int, span: int, device: int = 0, stream: int = 0,
                   pg=None, **overrides) -> hetpipe.Context:
    """Collective: context for `rank` of a distributed placement (world G, VW
    span k; include/hetpipe.h hp_config.vw_span). Rank 0 draws the barrier
    communicator id; IPC handles of every rank's arena are all-gathered with
    torch.distributed (process group `pg`, default group), then hp_connect maps
    the peers. After this every rank must drive the same protocol calls."""
    import torch.distributed as dist
    _nccl_hint()
    c = hetpipe.config_from(cfg, world=world, rank=rank, vw_span=span, device=device,
                            stream=stream or None, **overrides)
    ctx = hetpipe.Context(c)
    ids = [hetpipe.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0, group=pg)
    handles = [None] * world
    dist.all_gather_object(handles, ctx.ipc_handle(), group=pg)
    ctx.connect(handles, ids[0])
    return ctx


def symmetric_context(cfg, rank: int, world: int, span: int, device: int = 0, stream: int = 0,
                      pg=None, **overrides):
    """Collective: like placed_context, but the arena is a torch symmetric-memory
    allocation (device memory plumbing: torch maps every peer's arena and, on
    NVSwitch systems, a multicast mapping of all of them), handed to the library
    through hp_config.arena + hp_connect_symmetric. Needed for HP_XPORT_NVLS.
    Returns (ctx, keepalive): keep `keepalive` referenced while ctx lives."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    _nccl_hint()
    c = hetpipe.config_from(cfg, world=world, rank=rank, vw_span=span, device=device,
                            stream=stream or None, **overrides)
    nbytes = hetpipe.arena_bytes(c)
    sizes = [None] * world
    dist.all_gather_object(sizes, nbytes, group=pg)
    nbytes = max(sizes)                  # one size for the symmetric allocation
    buf = symm.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    h = symm.rendezvous(buf, pg if pg is not None else dist.group.WORLD)
    c.arena = buf.data_ptr()
    ctx = hetpipe.Context(c)
    ids = [hetpipe.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0, group=pg)
    mc = int(getattr(h, "multicast_ptr", 0) or 0)
    ctx.connect_symmetric([int(p) for p in h.buffer_ptrs], mc, ids[0])
    return ctx, (buf, h)

"""Multi-GPU plumbing (torch.distributed): packet sharding and the update-delta broadcast.

Packets partition trivially (each is classified independently), so every rank holds a
replica of the model and the tables and classifies its own shard -- no data-path collective.
The one exchange step is a rule update: rank 0 (the update leader) plans the insert/delete
ops on its host mirror (tang_update_plan), and the resulting word delta is broadcast --
NCCL over NVLink when the group is NCCL, landing directly in device memory -- and applied
in place on every rank's device tables (tang_apply_delta_async), ordered on the stream that
classifies, so every rank switches to table epoch e+1 at the same batch index.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import tang as T


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, end) of n packets owned by `rank` (sizes differ by at most one)."""
    q, r = divmod(n, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def broadcast_update(ctx: T.Ctx, ops, group=None, stream=None, mirror: bool = True):
    """Apply `ops` (meaningful on rank 0 only) on every rank of `group`.

    Returns (per-op status on rank 0 / None elsewhere, delta size in bytes).  With an NCCL
    group the delta travels device to device; with gloo it travels through host memory
    (CPU tests).  `mirror` keeps followers' host mirrors in step (checksums comparable)."""
    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    status, delta = None, b""
    if rank == 0:
        status, delta = ctx.update_plan(ops)
    ln = torch.tensor([len(delta)], dtype=torch.int64, device=dev)
    dist.broadcast(ln, 0, group=group)
    nbytes = int(ln.item())
    buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    if rank == 0 and nbytes:
        buf[:nbytes].copy_(torch.frombuffer(bytearray(delta), dtype=torch.uint8))
    if nbytes:
        dist.broadcast(buf, 0, group=group)
    if nccl:
        if nbytes:
            ctx.apply_delta_async(buf, nbytes, stream)
        if rank != 0 and mirror and nbytes:
            ctx.apply_delta_host(bytes(buf[:nbytes].cpu().numpy()))
    elif rank != 0 and nbytes:
        ctx.apply_delta_host(bytes(buf[:nbytes].numpy()))
    return status, nbytes


def checksums_agree(ctx: T.Ctx, group=None) -> bool:
    """All ranks hold byte-identical table mirrors (FNV-1a of every table)."""
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    c = torch.tensor([ctx.stats()["checksum"] & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(c) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, c, group=group)
    return all(int(o.item()) == int(c.item()) for o in out)


def max_over_ranks(x: float, group=None) -> float:
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())

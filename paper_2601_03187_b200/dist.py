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
            # the broadcast completed on torch's current stream: order the apply after it, and keep
            # buf alive (caching allocator) until the apply on `stream` has read it
            cur = torch.cuda.current_stream(dev)
            st = stream if stream is not None else cur
            if st.cuda_stream != cur.cuda_stream:
                st.wait_stream(cur)
            ctx.apply_delta_async(buf, nbytes, st)
            buf.record_stream(st)
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


def numa_cpus(device_index: int):
    """CPUs on the NUMA node closest to GPU `device_index` (NVML), or None if NVML cannot say."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)      # bitmask of ideal CPUs, 64 CPUs per word
    except Exception:
        return None
    cpus = [64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1]
    return cpus or None


def bind_numa_local(device_index: int):
    """Pin this rank's host thread to the CPUs of its GPU's NUMA node before the ctx allocates its
    pinned rings, so the rings' pages are placed (first touch) on that node and the streaming
    thread stays there (each rank reads its own NUMA-local ring).  Returns the CPU
    list, or None when NVML or the affinity call is unavailable (the rank then runs unpinned)."""
    import os
    cpus = numa_cpus(device_index)
    if not cpus:
        return None
    try:
        os.sched_setaffinity(0, cpus)
    except OSError:
        return None
    return cpus


def window_digests(ctx: T.Ctx, group=None, stream=None) -> torch.Tensor:
    """Every rank's table digest after an update window, all-gathered: int64 [world], rank order.
    NCCL: the digest of the DEVICE tables (tang_table_digest_async on `stream`, 8 bytes per rank
    over NVLink, no host synchronisation -- compare after the timed region); gloo: the host
    mirror's digest (CPU tests).  Equal entries = every replica applied the same deltas."""
    nccl = dist.get_backend(group) == "nccl"
    world = dist.get_world_size(group)
    if nccl:
        dev = torch.device("cuda", torch.cuda.current_device())
        d = torch.zeros(1, dtype=torch.int64, device=dev)
        cur = torch.cuda.current_stream(dev)
        st = stream if stream is not None else cur
        ctx.digest_async(d, st)
        if st.cuda_stream != cur.cuda_stream:
            cur.wait_stream(st)
    else:
        v = ctx.mirror_digest()
        d = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v], dtype=torch.int64)
    out = torch.zeros(world, dtype=torch.int64, device=d.device)
    dist.all_gather_into_tensor(out, d, group=group)
    return out

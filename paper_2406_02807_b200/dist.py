"""Multi-GPU plumbing: one process per GPU, query batches sharded,
tree replicated by one NCCL broadcast of its device slab, one all-reduce of
the counters at the end.  The query path itself has no data-path collective.

The helpers only use torch.distributed collectives, so the host logic runs
with the ``gloo`` backend on CPU tensors as well (tests/test_dist_gloo.py).
"""

from __future__ import annotations

__all__ = ["shard_range", "broadcast_bytes", "replicate_tree", "reduce_counters"]


def shard_range(n: int, world: int, rank: int, align: int = 32) -> tuple[int, int]:
    """Contiguous [start, stop) of rank's share of n items: ceil(n / world)
    rounded up to a multiple of ``align`` (32 spheres = one mask word, or
    32 groups x lane width), the last ranks take the remainder."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    if align < 1:
        raise ValueError("align must be >= 1")
    per = -(-n // world)
    per = -(-per // align) * align
    start = min(n, rank * per)
    stop = min(n, start + per)
    return start, stop


def broadcast_bytes(buf, src: int = 0, group=None, device=None):
    """Broadcast a uint8 tensor of unknown size from ``src``; other ranks pass
    None and receive a new tensor on ``device`` (CPU for gloo)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    size = torch.zeros(1, dtype=torch.int64, device=dev)
    if rank == src:
        size[0] = buf.numel()
    dist.broadcast(size, src, group=group)
    if rank != src:
        buf = torch.empty(int(size.item()), dtype=torch.uint8, device=dev)
    dist.broadcast(buf, src, group=group)
    return buf


def replicate_tree(tree, src: int = 0, group=None, device=None):
    """Broadcast ``tree`` (a Capt on rank ``src``; ignored elsewhere) to every
    rank of ``group`` over NCCL and return each rank's local replica."""
    import torch
    import torch.distributed as dist

    from .tree import Capt

    rank = dist.get_rank(group)
    if device is None:
        device = torch.cuda.current_device()
    dev = torch.device("cuda", device)
    slab = tree.slab_tensor() if rank == src else None
    slab = broadcast_bytes(slab, src, group, dev)
    if rank == src:
        return tree
    torch.cuda.synchronize(dev)
    return Capt.from_slab(slab, device=device, adopt=True)


def reduce_counters(counters, group=None):
    """Sum the per-rank counters (collisions, boundary, scanned, fixups,
    rejections, reserved) over the group, in place; returns the tensor."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters

"""Multi-GPU plumbing: one process per GPU, the collection sharded by set.

SURVEY 8(e): the (query, set) pairs are independent, so the collection is
split into contiguous set ranges, one per rank; the query sketches are
broadcast from rank 0 (NCCL over NVLink); every rank scores its shard with
set IDs offset by its shard base; the per-shard hit lists are gathered to
rank 0 (all_gather of counts, then an all_gather of the records padded to
the largest count) and merged there by `topk_or_threshold_results`.

Everything here works on any torch.distributed backend: NCCL with CUDA
tensors on the GPU box; gloo with CPU tensors in the CPU tests, or with CUDA
tensors staged through host memory (`bench.py --dist-backend gloo` runs two
ranks on one GPU that way).
"""
from __future__ import annotations

import numpy as np

HIT_BYTES = 20


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of set indices owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def _host_staged(t, group=None) -> bool:
    """gloo moves CPU tensors only: CUDA tensors are staged through host memory."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def broadcast_tensors(tensors, src: int = 0, group=None):
    """Broadcast a list of tensors (shapes already agreed) from `src`."""
    import torch.distributed as dist
    for t in tensors:
        if t is None:
            continue
        if _host_staged(t, group):
            h = t.cpu()
            dist.broadcast(h, src=src, group=group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=src, group=group)


def all_gather(outs, t, group=None):
    import torch
    import torch.distributed as dist
    if _host_staged(t, group):
        hs = [torch.empty_like(o, device="cpu") for o in outs]
        dist.all_gather(hs, t.cpu(), group=group)
        for o, h in zip(outs, hs):
            o.copy_(h)
    else:
        dist.all_gather(outs, t, group=group)


def gather_hits(hits_u8, count: int, group=None):
    """Gather per-rank hit records (uint8 tensor holding >= count*20 bytes) to
    every rank (all_gather: NCCL has no gatherv).  Returns (concatenated
    uint8 tensor of all records in rank order, per-rank counts)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = hits_u8.device
    cnt = torch.tensor([count], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(counts) if counts else 0
    if mx == 0:
        return torch.zeros((0,), dtype=torch.uint8, device=dev), counts
    pad = torch.zeros((mx * HIT_BYTES,), dtype=torch.uint8, device=dev)
    pad[: count * HIT_BYTES] = hits_u8[: count * HIT_BYTES]
    bufs = [torch.empty_like(pad) for _ in range(world)]
    all_gather(bufs, pad, group=group)
    out = torch.cat([b[: c * HIT_BYTES] for b, c in zip(bufs, counts)])
    return out, counts


def max_over_ranks(x: float, group=None, device="cpu") -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if _host_staged(t, group):
        t = t.cpu()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def records_from_bytes(u8) -> np.ndarray:
    from . import HIT_DTYPE
    return u8.cpu().numpy().view(HIT_DTYPE)


def merge_threshold_records(recs: np.ndarray) -> np.ndarray:
    """Host reference of the rank-0 merge for threshold lists: the gathered
    records in (query, set_id) order (what topk_or_threshold_results does on
    the device).  Used by the CPU tests of the sharded path."""
    order = np.lexsort((recs["set_id"], recs["query"]))
    return recs[order]

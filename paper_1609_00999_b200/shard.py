"""Shard / launch layer.

Arrays shard trivially: rank r of W owns the contiguous slice
[floor(r n / W), floor((r+1) n / W)) of every element-wise problem, inputs are
generated from the GLOBAL index (so results do not depend on W), and the only
collective is one SUM all-reduce of the per-rank checksum partials after the
timed region (plus a MAX all-reduce of elapsed times for box timing).  There is
no exchange step on the data path, so none is invented.

Backend-agnostic: works with "nccl" (CUDA tensors, one process per GPU) and
"gloo" (CPU tensors; used by the world_size-2 CPU tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world():
    """(rank, local_rank, world_size) from the torchrun environment (defaults: 0, 0, 1)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def slice_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice of rank `rank`: [floor(r n / W), floor((r+1) n / W))."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard request")
    return (rank * n) // world, ((rank + 1) * n) // world


def _device_for(group=None):
    backend = dist.get_backend(group) if dist.is_initialized() else "gloo"
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def combine_checksums(local_sums, P, group=None):
    """All-reduce SUM of per-rank uint64 partial sums, then reduce mod P.

    `local_sums` is a list of Python ints (one per prime / problem) or a single
    int; each partial is reduced mod P first so the W-way sum stays < W*P."""
    single = not isinstance(local_sums, (list, tuple))
    sums = [local_sums] if single else list(local_sums)
    Ps = [P] * len(sums) if not isinstance(P, (list, tuple)) else list(P)
    vals = torch.tensor([int(s) % int(p) for s, p in zip(sums, Ps)], dtype=torch.int64,
                        device=_device_for(group))
    if dist.is_initialized():
        dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
    out = [int(v) % int(p) for v, p in zip(vals.tolist(), Ps)]
    return out[0] if single else out


def max_over_ranks(x: float, group=None) -> float:
    """Box timing: the MAX of a per-rank float over all ranks."""
    if not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def barrier(group=None) -> None:
    if dist.is_initialized():
        if dist.get_backend(group) == "nccl":
            dist.barrier(group=group, device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier(group=group)

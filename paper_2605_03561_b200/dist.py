"""Rank sharding for multi-GPU queries (one process per GPU).

Traces shard by rank into contiguous ranges; the query's
summaries travel over NCCL (psg_comm_init) or, through a host reducer, over
any torch.distributed process group (psg_comm_init_host) — gloo on CPU, or
several ranks sharing one GPU.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) of n traces owned by `rank` of `world` (sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * n // world, (rank + 1) * n // world


def node_aligned_ranges(node_of_trace, world: int, weights=None) -> list[tuple[int, int]]:
    """Contiguous shard ranges balanced by `weights` (events per trace; 1 by
    default) whose edges fall on node boundaries, so per-node sums (node means)
    never straddle two ranks.  node_of_trace must be non-decreasing."""
    node = np.asarray(node_of_trace)
    n = len(node)
    if n and np.any(np.diff(node) < 0):
        raise ValueError("node_of_trace must be non-decreasing")
    w = np.ones(n, np.float64) if weights is None else np.asarray(weights, np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    starts = np.flatnonzero(np.concatenate([[True], node[1:] != node[:-1]])) if n else np.zeros(0, int)
    edges = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        # the node start closest to the target weight, never moving backwards
        i = int(np.argmin(np.abs(cum[starts] - target))) if len(starts) else 0
        e = int(starts[i]) if len(starts) else 0
        edges.append(max(e, edges[-1]))
    edges.append(n)
    return [(edges[r], edges[r + 1]) for r in range(world)]


def torch_reducer(group=None):
    """A host reducer over a torch.distributed process group: reduces a
    uint64/float64 numpy array in place (uint64 travels as int64: sums wrap
    identically; min/max flip the sign bit around the exchange so that they
    compare in unsigned order for every value)."""
    import torch
    import torch.distributed as dist

    ops = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}

    def reduce(arr: np.ndarray, op: str) -> None:
        if arr.dtype == np.uint64:
            # min / max in unsigned order: flip the sign bit so that the signed
            # int64 comparison orders like uint64 (sums wrap identically)
            flip = op in ("min", "max")
            if flip:
                arr ^= np.uint64(1 << 63)
            t = torch.from_numpy(arr.view(np.int64))
            dist.all_reduce(t, op=ops[op], group=group)  # in place: t shares arr's memory
            if flip:
                arr ^= np.uint64(1 << 63)
            return
        t = torch.from_numpy(arr)
        dist.all_reduce(t, op=ops[op], group=group)  # in place: t shares arr's memory
    return reduce

"""Replica sharding of colourings across ranks (SURVEY §8(e) "R").

Colouring j is a pure function of (seed, j, v) (sg2v.h, sg2v_count), so the N
colourings of an estimate (Alg. 1 line 3) shard across G ranks without
any communication during the DP: rank r runs j = iter_offset + r + G·t.  The one
exchange of the path is the end: an all-reduce (sum) of the per-colouring
counts, zero-padded outside each rank's slots, which is exact because every
slot has exactly one contributor.  torch.distributed carries it (NCCL on B200,
gloo on CPU for the tests).
"""
from __future__ import annotations

import math

import numpy as np


def shard(n_iter: int, rank: int, world: int, iter_offset: int = 0):
    """(first colouring, stride, how many) owned by `rank`."""
    if n_iter < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    mine = max(0, math.ceil((n_iter - rank) / world))
    return iter_offset + rank, world, mine


def gather_counts(local: np.ndarray, n_iter: int, rank: int, world: int, precision: str, device=None, group=None):
    """All-reduce the rank-local per-colouring counts into the full [n_iter] vector."""
    import torch
    import torch.distributed as dist

    u64 = precision == "u64"
    dtype = torch.int64 if u64 else torch.float64
    full = torch.zeros(n_iter, dtype=dtype, device=device)
    if len(local):
        vals = torch.from_numpy(local.view(np.int64) if u64 else local.astype(np.float64))
        full[rank::world] = vals.to(full.device)
    if world > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    out = full.cpu().numpy()
    return out.view(np.uint64) if u64 else out


def count_replicated(graph, tmpl, n_iter: int, seed: int, precision: str = "f32", iter_offset: int = 0,
                     rank: int = 0, world: int = 1, count_fn=None, device=None, group=None, **kw):
    """Estimate over n_iter colourings split across `world` ranks.

    count_fn(graph, tmpl, n, seed, precision, iter_offset, iter_stride, **kw) ->
    per-colouring counts (default: the CUDA path, paper_2009_11665_b200.count).
    Returns (estimate, full per-colouring vector) on every rank.
    """
    if count_fn is None:
        from .sg2v import count as _count

        def count_fn(g, t, n, s, p, off, stride, **k2):
            return _count(g, t, n_iter=n, seed=s, precision=p, iter_offset=off, iter_stride=stride, **k2)[1]

    first, stride, mine = shard(n_iter, rank, world, iter_offset)
    if mine:
        local = np.asarray(count_fn(graph, tmpl, mine, seed, precision, first, stride, **kw))
    else:
        local = np.zeros(0, dtype=np.uint64 if precision == "u64" else np.float64)
    full = gather_counts(local, n_iter, rank, world, precision, device=device, group=group)
    if precision == "u64":
        return float("nan"), full
    if not n_iter:
        return float("nan"), full
    from .sg2v import estimate  # a7 (mean / (P·α)) runs in the C ABI: sg2v_estimate
    return estimate(tmpl, full), full

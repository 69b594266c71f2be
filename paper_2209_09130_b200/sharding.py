"""Batch sharding across GPUs: one process per GPU, independent engine replicas.

Inference shards naturally by sequence (the reference runs sequences
independently, encoder.py:472), so multi-GPU is data-parallel with no
collective on the data path:
  * ``partition_by_tokens`` splits a packed batch into contiguous per-rank shards
    balanced by token count (varlen batches, config C3/C5);
  * ``max_over_ranks`` turns per-rank device times into the job time;
  * ``gather_rows`` is the optional output gather (rank 0 receives every shard's
    logits) — bytes, not bandwidth: it is not on the timed path.
Works with the ``nccl`` backend on B200s and ``gloo`` on CPU (tests).
"""

from __future__ import annotations

import numpy as np


def partition_by_tokens(lengths, world: int) -> list:
    """Contiguous shards [(s0, s1), ...] of len(lengths) sequences, one per rank, with
    token counts as equal as a greedy prefix split allows (every rank gets >= 1 sequence
    when there are at least `world` sequences)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    n = len(lengths)
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.concatenate([[0], np.cumsum(lengths)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        cut = int(np.searchsorted(cum, target, side="left"))
        if cut > 0 and abs(cum[cut - 1] - target) <= abs(cum[cut] - target):
            cut -= 1
        lo = bounds[-1] + (1 if n - bounds[-1] > world - r else 0)
        hi = n - (world - r)
        bounds.append(int(min(max(cut, lo), max(hi, lo))))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(value: float, device=None) -> float:
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: np.ndarray):
    """Rank 0 gets the concatenation of every rank's rows (None elsewhere)."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return local
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, local)
    return np.concatenate(parts, axis=0) if dist.get_rank() == 0 else None

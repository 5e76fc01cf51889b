"""Data-parallel plumbing: utterances are independent, so ranks
take disjoint shards and the only collective is one all-reduce of the 5
float64 totals {Σ loss, Σ N_b, Σ logZ_num, Σ logZ_den, n_bad} per step.

Sharding is longest-processing-time-first over cost N_b · (nnz_den + nnz_num,b),
mirroring the paper's length-bucketed batches; within a rank the
shard is ordered longest first.
"""
from __future__ import annotations

import heapq
from typing import List, Sequence

import numpy as np


def lpt_shard(costs: Sequence[float], world: int) -> List[np.ndarray]:
    """Greedy LPT: largest cost first onto the least-loaded rank (ties → lowest rank).
    Returns, per rank, the utterance indices ordered longest first."""
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    shards = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [np.array(s, dtype=np.int64) for s in shards]


def utterance_costs(lengths, num_nnz, den_nnz: int) -> np.ndarray:
    return np.asarray(lengths, np.float64) * (float(den_nnz) + np.asarray(num_nnz, np.float64))


def allreduce_totals(totals):
    """Sum the 5 per-rank totals over the default process group (NCCL on the
    current stream for CUDA tensors, gloo for CPU tensors)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(totals)
    return totals

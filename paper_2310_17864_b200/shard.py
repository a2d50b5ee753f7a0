"""Length-balanced utterance sharding across GPUs.

Utterances are independent, so the batch is partitioned with no data-path
collective: longest-processing-time-first (LPT) on cost ∝ len_b (V and beam
are constant per decoder), each utterance to the currently least-loaded rank.
Results are reassembled on the host in original index order.
"""

from __future__ import annotations

import heapq

import numpy as np


def lpt_shards(lens, n_ranks: int) -> list[np.ndarray]:
    """Split utterance indices into ``n_ranks`` shards with balanced Σ len.

    Deterministic: ties in length break by index, ties in load by rank.  Each
    shard's indices are returned in ascending order.
    """
    lens = np.asarray(lens, dtype=np.int64)
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    order = sorted(range(len(lens)), key=lambda i: (-int(lens[i]), i))
    heap = [(0, r) for r in range(n_ranks)]
    shards: list[list[int]] = [[] for _ in range(n_ranks)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + max(int(lens[i]), 1), r))
    return [np.array(sorted(s), dtype=np.int64) for s in shards]


def balanced_ranges(lens, n_parts: int) -> list[tuple[int, int]]:
    """Split ``range(len(lens))`` into ``n_parts`` consecutive ranges with
    balanced Σ max(len, 1): part k ends at the first index whose prefix load
    reaches (k+1)/n of the total.  Consecutive ranges are views of a [B, T, V]
    batch (no host gather), and each device's kernel orders its own range
    longest-first, so only the per-range sums need balancing.  Empty ranges
    appear when n_parts > len(lens)."""
    lens = np.maximum(np.asarray(lens, dtype=np.int64), 1)
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    B = len(lens)
    pre = np.concatenate([[0], np.cumsum(lens)])
    total = int(pre[-1])
    cuts = [0]
    for k in range(1, n_parts):
        # smallest b with pre[b] >= k * total / n, rounded to the nearer side
        target = total * k / n_parts
        b = int(np.searchsorted(pre, target, side="left"))
        if 0 < b <= B and target - pre[b - 1] < pre[b] - target:
            b -= 1
        cuts.append(min(max(b, cuts[-1]), B))
    cuts.append(B)
    return [(cuts[k], cuts[k + 1]) for k in range(n_parts)]


def merge_shards(shards: list[np.ndarray], per_rank_results: list[list], n_total: int) -> list:
    """Reassemble per-rank result lists (in shard index order) into batch order."""
    out = [None] * n_total
    for idx, res in zip(shards, per_rank_results):
        if len(idx) != len(res):
            raise ValueError("shard/result length mismatch")
        for i, r in zip(idx.tolist(), res):
            out[i] = r
    if any(r is None for r in out):
        raise ValueError("shards do not cover the batch")
    return out

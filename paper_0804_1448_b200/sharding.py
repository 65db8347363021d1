"""Reference-set sharding plan for multi-GPU searches.

Rank r of N owns the contiguous reference range [shard_bounds(m, N, r)); its
device search returns raw keys with GLOBAL indices (index_base = lo), the
per-rank n x k lists are all-gathered into a [N, n, k] buffer (rank-major) and
merged on device (knn_b200_merge_device).  Because every rank's list is the
exact top-k of a disjoint range under the (key, index) order, the merged table
is bitwise identical to a single-device search over all of R.
"""
from __future__ import annotations


def shard_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced, covering ranges: sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} out of range for world {world}")
    return rank * m // world, (rank + 1) * m // world


def check_shardable(m: int, world: int, k: int) -> None:
    """Every shard must hold >= k references so each rank returns a full list."""
    smallest = m // world
    if smallest < k:
        raise ValueError(f"reference-sharded search needs m/world >= k ({m}/{world} < {k})")

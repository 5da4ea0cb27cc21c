"""Launcher-side partition of the independent B*H head grid.

Every (b,h) head is an independent reference call: ranks own contiguous head ranges and run the
same kernels on their shard; there is NO collective on the hot path.  torch.distributed is only used by
bench.py / tests to gather outputs or checksums for verification.
"""
from __future__ import annotations


def shard_range(total_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Same arithmetic as ba_shard_range in the C ABI (first total%world ranks own one extra head)."""
    if total_heads < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: need total >= 0 and 0 <= rank < world")
    base, rem = divmod(total_heads, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def shard_heads(t, world: int, rank: int):
    """Slice a [B,H,...] tensor down to this rank's heads, flattened to [1, heads_local, ...]."""
    B, H = t.shape[0], t.shape[1]
    b, e = shard_range(B * H, world, rank)
    return t.reshape(1, B * H, *t.shape[2:])[:, b:e]

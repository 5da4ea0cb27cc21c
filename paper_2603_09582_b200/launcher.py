"""Launcher: one process per GPU, the independent (batch, head) grid sharded across ranks.

Every (b,h) head is an independent reference call: mu is per head (quantize.cpp:16-23), the bias is per call.
Rank r of `world` owns a contiguous range of the flattened B*H grid (ba_shard_range / shard_range) -- or, with
shard_units, a contiguous range of (head, 256-query-row block) units, which may split a head -- and runs the same
kernels on its shard.  There is NO collective on the hot path; torch.distributed (NCCL on GPUs, gloo in the CPU tests) is
used only by `gather` to collect the outputs for verification, outside any timed region.

    sh = ShardedBinaryAttention()                  # RANK / WORLD_SIZE / LOCAL_RANK from the environment (torchrun)
    Ql, Kl, Vl, bl = sh.shard(Q, K, V, bias)       # this rank's heads (views where the shard allows it)
    Ol = sh.forward(Ql, Kl, Vl, bl)                # K1 + K2 on this rank's GPU
    O = sh.gather(Ol, B, H)                        # [B,H,N,d] on every rank (verification only)
"""
from __future__ import annotations

import os


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Same arithmetic as ba_shard_range / ba_shard_units in the C ABI (the first total % world ranks own one extra item)."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: need total >= 0 and 0 <= rank < world")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def shard_heads(t, world: int, rank: int):
    """Slice a [B,H,...] tensor down to this rank's heads, flattened to [1, heads_local, ...]."""
    B, H = t.shape[0], t.shape[1]
    b, e = shard_range(B * H, world, rank)
    return t.reshape(1, B * H, *t.shape[2:])[:, b:e]


def shard_plan(B: int, H: int, world: int, rank: int) -> dict:
    """How rank `rank` slices a [B,H,N,d] batch: whole batch elements when B divides evenly (the bias table stays [H,N,N]),
    else a contiguous range of the flattened head grid as [1, heads, N, d] with one bias table per local head."""
    if B % world == 0:
        b, e = shard_range(B, world, rank)
        return {"mode": "batch", "begin": b * H, "end": e * H, "b0": b, "b1": e}
    b, e = shard_range(B * H, world, rank)
    return {"mode": "heads", "begin": b, "end": e}


def shard_units(B: int, H: int, N: int, world: int, rank: int) -> tuple[int, int]:
    """ba_shard_units: contiguous range of the B*H*ceil(N/256) (head, 256-query-row block) units owned by `rank`; pass it to
    BinaryAttention.forward(..., units=...) on tensors that hold every head the range touches."""
    return shard_range(B * H * ((N + 255) // 256), world, rank)


class ShardedBinaryAttention:
    """Per-GPU launcher for a sharded BinaryAttention forward (see the module docstring)."""

    def __init__(self, rank: int | None = None, world: int | None = None, local_rank: int | None = None, device=None):
        self.rank = int(os.environ.get("RANK", "0")) if rank is None else rank
        self.world = int(os.environ.get("WORLD_SIZE", "1")) if world is None else world
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0")) if local_rank is None else local_rank
        self._ba = None
        self._device = device

    @property
    def ba(self):
        if self._ba is None:
            import torch
            from .api import BinaryAttention
            dev = self._device or torch.device("cuda", self.local_rank)
            self._ba = BinaryAttention(dev)
        return self._ba

    def plan(self, B: int, H: int) -> dict:
        return shard_plan(B, H, self.world, self.rank)

    def shard(self, Q, K, V, bias=None):
        """This rank's part of a full [B,H,N,d] batch and of its dense bias [1|H,N,N] (None passes through)."""
        B, H = Q.shape[0], Q.shape[1]
        pl = self.plan(B, H)
        if pl["mode"] == "batch":
            sl = slice(pl["b0"], pl["b1"])
            return Q[sl], K[sl], V[sl], bias
        cut = lambda t: t.reshape(1, B * H, *t.shape[2:])[:, pl["begin"]:pl["end"]]
        bl = bias
        if bias is not None and bias.dim() == 3 and bias.shape[0] == H:
            idx = [g % H for g in range(pl["begin"], pl["end"])]
            contiguous = all(idx[i] + 1 == idx[i + 1] for i in range(len(idx) - 1))
            bl = bias[idx[0]:idx[-1] + 1] if idx and contiguous else bias[idx]  # a view when the range does not wrap
        return cut(Q), cut(K), cut(V), bl

    def forward(self, Q, K, V, bias=None, scale=None, kernel="auto", out_dtype=None):
        import torch
        out_dtype = out_dtype or torch.float32
        if Q.shape[1] == 0:
            return torch.empty(Q.shape, dtype=out_dtype, device=Q.device)
        return self.ba.forward(Q, K, V, bias, scale, kernel=kernel, out_dtype=out_dtype)

    def forward_units(self, Q, K, V, bias=None, scale=None, kernel="auto", out=None, out_dtype=None):
        """Unit-sharded forward on the FULL [B,H,N,d] tensors (resident on every rank): this rank computes its (head, 256-row
        block) units only; rows of other ranks' units stay zero in the returned tensor (sum or gather to combine)."""
        B, H, N = Q.shape[0], Q.shape[1], Q.shape[2]
        import torch
        return self.ba.forward(Q, K, V, bias, scale, kernel=kernel, units=shard_units(B, H, N, self.world, self.rank), out=out,
                               out_dtype=out_dtype or torch.float32)

    def gather(self, O_local, B: int, H: int):
        """All ranks' outputs as one [B,H,N,d] tensor (all_gather of equal-size padded shards; verification only)."""
        import torch
        import torch.distributed as dist
        N, d = O_local.shape[-2], O_local.shape[-1]
        flat = O_local.reshape(-1, N, d)
        if self.world == 1:
            return flat.reshape(B, H, N, d)
        sizes = [shard_plan(B, H, self.world, r) for r in range(self.world)]
        most = max(s["end"] - s["begin"] for s in sizes)
        pad = torch.zeros((most, N, d), dtype=flat.dtype, device=flat.device)
        pad[:flat.shape[0]] = flat
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad)
        return torch.cat([o[:s["end"] - s["begin"]] for o, s in zip(out, sizes)]).reshape(B, H, N, d)

"""Multi-GPU partitioning of the PSA forward.

Work units are (batch, head): heads are independent in the reference (the per-head loop of
pkg/src/pyrattn/pipeline.py:363-369 carries no state across heads), so each rank owns whole KV
heads together with their GQA query-head group and runs the single-GPU path on them — no
per-call collective. ``gather_outputs`` is the optional NCCL gather of O onto one rank, used
only when the caller wants the full output on one device (timed separately by bench.py).
"""

from __future__ import annotations

import math

import torch


def shard_heads(hq: int, hkv: int, world: int, rank: int) -> tuple[list, list]:
    """(query heads, kv heads) owned by ``rank``: contiguous KV-head ranges, query heads follow
    their KV head (q head h reads kv head h // (hq // hkv))."""
    if hq % hkv:
        raise ValueError(f"query heads {hq} not a multiple of kv heads {hkv}")
    group = hq // hkv
    per = math.ceil(hkv / world)
    kv = list(range(rank * per, min(hkv, (rank + 1) * per)))
    q = [h for hk in kv for h in range(hk * group, (hk + 1) * group)]
    return q, kv


def gather_outputs(out_local: torch.Tensor, hq: int, hkv: int, dst: int = 0, group=None):
    """Gather per-rank [B, h_local, N, d] outputs into [B, hq, N, d] on rank ``dst`` (None on
    other ranks). Shards can be uneven, so every rank pads to the largest shard and the
    destination strips the padding. Works with the NCCL (GPU) and gloo (CPU) backends."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, _, N, d = out_local.shape
    sizes = [len(shard_heads(hq, hkv, world, r)[0]) for r in range(world)]
    pad = max(sizes)
    buf = out_local.new_zeros((B, pad, N, d))
    buf[:, : out_local.shape[1]] = out_local
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    if dist.get_backend(group) == "nccl":
        # NCCL has no gather: all_gather into the destination buffers (others discard)
        parts_all = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts_all, buf, group=group)
        parts = parts_all if rank == dst else None
    else:
        dist.gather(buf, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([p[:, :s] for p, s in zip(parts, sizes)], dim=1)

"""Multi-GPU partitioning of the PSA forward.

Heads are independent in the reference (the per-head loop of pkg/src/pyrattn/pipeline.py:363-369
carries no state across heads), so each rank owns a contiguous, balanced range of QUERY heads
(floor/ceil of hq / world) and runs the single-GPU path on them, with no per-call collective. A
rank reads every KV head its query heads use; under GQA a KV head whose query group is split
between two ranks is read (and its pyramid built) on both, which is cheap next to the query work.
``shard_segments`` cuts a rank's range into calls with uniform GQA grouping (at most a partial
group, a run of whole groups and another partial group). ``gather_outputs`` is the optional NCCL
gather of O onto one rank, used only when the caller wants the full output on one device.
"""

from __future__ import annotations

import torch


def _check(hq: int, hkv: int, world: int, rank: int) -> int:
    if hq % hkv:
        raise ValueError(f"query heads {hq} not a multiple of kv heads {hkv}")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return hq // hkv


def shard_heads(hq: int, hkv: int, world: int, rank: int) -> tuple[list, list]:
    """(query heads, kv heads) of ``rank``: a balanced contiguous query-head range and the KV
    heads it reads (q head h reads kv head h // (hq // hkv))."""
    group = _check(hq, hkv, world, rank)
    q = list(range(rank * hq // world, (rank + 1) * hq // world))
    kv = sorted({h // group for h in q})
    return q, kv


def shard_segments(hq: int, hkv: int, world: int, rank: int) -> list:
    """The rank's query heads as calls with uniform GQA: [(q_lo, q_hi, kv_lo, kv_hi)], each
    with (q_hi - q_lo) a multiple of (kv_hi - kv_lo) and q head h of the call reading kv head
    kv_lo + (h - q_lo) // ((q_hi - q_lo) // (kv_hi - kv_lo))."""
    group = _check(hq, hkv, world, rank)
    lo, hi = rank * hq // world, (rank + 1) * hq // world
    segs = []
    while lo < hi:
        kv = lo // group
        if lo % group or hi < (kv + 1) * group:  # partial group of one kv head
            end = min(hi, (kv + 1) * group)
            segs.append((lo, end, kv, kv + 1))
            lo = end
        else:  # run of whole groups
            kv_end = hi // group
            segs.append((lo, kv_end * group, kv, kv_end))
            lo = kv_end * group
    return segs


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

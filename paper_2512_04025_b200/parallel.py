"""Multi-GPU partitioning of the PSA forward.

Heads are independent in the reference (the per-head loop of pkg/src/pyrattn/pipeline.py:363-369
carries no state across heads) and so are the query blocks of a head given its K/V
(pkg/src/pyrattn/attention.py:187; importance.py:52-132 and mask.py:128-151 work row by row). The
work unit is therefore (batch, query head, query-block set): every head is cut into ``parts``
equal-cost query-block sets, just enough that the units divide evenly over the ranks, and each
rank runs a contiguous run of units with no per-call collective. A rank builds the pyramid of
every KV head its units read (an HBM-cheap pass, repeated on the ranks that share a head).

Part shapes: without causal masking every query block costs about the same (the budget is per
row), so a part is a contiguous block range. Under causal masking block i sees ~(i + 1) blocks, so
blocks are dealt in zigzag pairs (i, n_q - 1 - i) of equal total cost.

``partition`` returns, per rank, the calls to make: (q_lo, q_hi, kv_lo, kv_hi, qblocks) with a
uniform GQA grouping inside each call and ``qblocks`` None for whole heads. ``gather_outputs`` is
the optional gather of O onto one rank (NCCL or gloo), used only when the caller wants the whole
output on one device.
"""

from __future__ import annotations

import math

import torch


def _check(hq: int, hkv: int, world: int, rank: int) -> int:
    if hq % hkv:
        raise ValueError(f"query heads {hq} not a multiple of kv heads {hkv}")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return hq // hkv


def shard_heads(hq: int, hkv: int, world: int, rank: int) -> tuple[list, list]:
    """(query heads, kv heads) of ``rank`` under whole-head sharding: a balanced contiguous
    query-head range and the KV heads it reads (q head h reads kv head h // (hq // hkv))."""
    group = _check(hq, hkv, world, rank)
    q = list(range(rank * hq // world, (rank + 1) * hq // world))
    kv = sorted({h // group for h in q})
    return q, kv


def shard_segments(hq: int, hkv: int, world: int, rank: int) -> list:
    """The rank's whole-head range as calls with uniform GQA: [(q_lo, q_hi, kv_lo, kv_hi)]."""
    _check(hq, hkv, world, rank)
    return head_range_segments(rank * hq // world, (rank + 1) * hq // world, hq, hkv)


def head_range_segments(lo: int, hi: int, hq: int, hkv: int) -> list:
    """Query heads [lo, hi) as calls with uniform GQA: [(q_lo, q_hi, kv_lo, kv_hi)], each with
    (q_hi - q_lo) a multiple of (kv_hi - kv_lo) and q head h of the call reading kv head
    kv_lo + (h - q_lo) // ((q_hi - q_lo) // (kv_hi - kv_lo))."""
    group = hq // hkv
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


def head_parts(hq: int, world: int) -> int:
    """Query-block parts per head so that hq * parts units divide evenly over ``world`` ranks."""
    return world // math.gcd(hq, world)


def part_blocks(n_q: int, parts: int, part: int, causal: bool) -> list:
    """Query blocks of part ``part`` of ``parts`` of one head (ascending): a contiguous range,
    or under causal masking a run of zigzag pairs (i, n_q - 1 - i)."""
    if not 0 <= part < parts or parts > n_q:
        raise ValueError(f"part {part} of {parts} for {n_q} query blocks")
    if not causal:
        return list(range(part * n_q // parts, (part + 1) * n_q // parts))
    pairs = (n_q + 1) // 2
    out = []
    for pi in range(part * pairs // parts, (part + 1) * pairs // parts):
        out.append(pi)
        if n_q - 1 - pi != pi:
            out.append(n_q - 1 - pi)
    return sorted(out)


def block_cost(blocks, n_q: int, causal: bool) -> float:
    """Relative attention cost of query blocks of one head: 1 per block, or (i + 1) / n_q per
    block under causal masking (block i sees ~i + 1 of the n_q key blocks)."""
    if not causal:
        return float(len(blocks))
    return float(sum(i + 1 for i in blocks)) / n_q * 2.0


def partition(hq: int, hkv: int, n_q: int, world: int, rank: int, causal: bool = False,
              parts: int | None = None) -> list:
    """Calls of ``rank``: [(q_lo, q_hi, kv_lo, kv_hi, qblocks)] covering its units. Whole heads
    (qblocks None) are grouped into uniform-GQA calls; a partial head is its own call with its
    query-block list (ascending)."""
    group = _check(hq, hkv, world, rank)
    parts = head_parts(hq, world) if parts is None else parts
    parts = max(1, min(parts, n_q))
    units = hq * parts
    u_lo, u_hi = rank * units // world, (rank + 1) * units // world
    calls = []
    u = u_lo
    while u < u_hi:
        h, pt = divmod(u, parts)
        if pt == 0 and u + parts <= u_hi:  # a run of whole heads [h, h_end)
            h_end = h + 1
            while (h_end + 1) * parts <= u_hi:
                h_end += 1
            for seg in head_range_segments(h, h_end, hq, hkv):
                calls.append(seg + (None,))
            u = h_end * parts
            continue
        last = min(u_hi, (h + 1) * parts)  # parts [pt, last - h * parts) of head h
        blocks = []
        for p_ in range(pt, last - h * parts):
            blocks += part_blocks(n_q, parts, p_, causal)
        calls.append((h, h + 1, h // group, h // group + 1, sorted(blocks)))
        u = last
    return calls


def rank_cost(calls, n_q: int, causal: bool) -> float:
    """Estimated attention cost of a rank's calls (in head-blocks)."""
    cost = 0.0
    for q_lo, q_hi, _, _, blocks in calls:
        blk = range(n_q) if blocks is None else blocks
        cost += (q_hi - q_lo) * block_cost(blk, n_q, causal)
    return cost


def gather_outputs(out_local: torch.Tensor, hq: int, hkv: int, dst: int = 0, group=None):
    """Gather per-rank [B, h_local, N, d] whole-head outputs (shard_heads) into [B, hq, N, d] on
    rank ``dst`` (None elsewhere). Shards can be uneven, so every rank pads to the largest shard
    and the destination strips the padding. dist.gather works on NCCL and gloo."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, _, N, d = out_local.shape
    sizes = [len(shard_heads(hq, hkv, world, r)[0]) for r in range(world)]
    pad = max(sizes)
    buf = out_local.new_zeros((B, pad, N, d))
    buf[:, : out_local.shape[1]] = out_local
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([p[:, :s] for p, s in zip(parts, sizes)], dim=1)


def gather_partitioned(pieces: list, hq: int, hkv: int, n_q: int, b_q: int, causal: bool,
                       dst: int = 0, group=None, parts: int | None = None):
    """Gather the outputs of ``partition`` calls onto rank ``dst`` as [B, hq, n_q * b_q, ...].
    ``pieces``: this rank's per-call outputs in call order, [B, heads, rows, *rest] with rows the
    call's query blocks (compact) or the whole sequence. Every rank flattens its pieces into one
    padded buffer; the destination places the rows by the (deterministic) partition."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    flat = torch.cat([p.reshape(-1) for p in pieces]) if pieces else None
    sizes = []
    ref = pieces[0]
    B, rest = ref.shape[0], tuple(ref.shape[3:])
    row_elems = math.prod(rest) if rest else 1
    for r in range(world):
        n = 0
        for q_lo, q_hi, _, _, blocks in partition(hq, hkv, n_q, world, r, causal, parts):
            nb = n_q if blocks is None else len(blocks)
            n += B * (q_hi - q_lo) * nb * b_q * row_elems
        sizes.append(n)
    buf = ref.new_zeros(max(sizes))
    if flat is not None:
        buf[: flat.numel()] = flat
    bufs = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    full = ref.new_empty((B, hq, n_q * b_q) + rest)
    for r in range(world):
        off = 0
        for q_lo, q_hi, _, _, blocks in partition(hq, hkv, n_q, world, r, causal, parts):
            blk = list(range(n_q)) if blocks is None else blocks
            n = B * (q_hi - q_lo) * len(blk) * b_q * row_elems
            part = bufs[r][off: off + n].view((B, q_hi - q_lo, len(blk), b_q) + rest)
            rows = full[:, q_lo:q_hi].view((B, q_hi - q_lo, n_q, b_q) + rest)
            rows[:, :, torch.tensor(blk, dtype=torch.long, device=rows.device)] = part
            off += n
    return full

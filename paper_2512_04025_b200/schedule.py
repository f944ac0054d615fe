"""Decoupled block-tile schedule: API parity with pkg/src/pyrattn/scheduler.py.

Drop-ins for Segment :24-35, ExecutionTile :38-45, TileSchedule :48-52, UtilizationStats :55-68,
build_schedule :71-126, _validate_schedule :129-200, execute_schedule :203-269,
utilization :272-282.

In this framework the attention kernel IS the decoupled block-tile executor: its producer warps
pack the selected pooled segments of several KV blocks into 128-row tiles on the fly (power-of-two
slots, level-major; psa_attention.cu). ``build_schedule`` reproduces the reference's greedy
in-order packing (a host-side plan description over the mask: index bookkeeping, no tensor
math) so callers and reports see the same tiles and utilisation as the reference;
``execute_schedule`` validates a schedule exactly as the reference does and runs it on the GPU
kernel (tiling changes only the chunking of the online softmax, scheduler.py:207-209);
``plan_utilization`` reports the fill of the tiles the kernel actually executes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ValidationError
from .layout import BlockLayout


@dataclass(frozen=True)
class Segment:
    """A contiguous slice of one pooled KV block inside a tile."""

    kv_block: int
    level: int
    row_start: int
    row_stop: int

    @property
    def rows(self) -> int:
        return self.row_stop - self.row_start


@dataclass(frozen=True)
class ExecutionTile:
    query_block: int
    segments: tuple

    @property
    def filled(self) -> int:
        return sum(s.rows for s in self.segments)


@dataclass(frozen=True)
class TileSchedule:
    tile_len: int
    tiles: tuple
    layout: BlockLayout


@dataclass(frozen=True)
class UtilizationStats:
    tiles: int
    useful_rows: int
    capacity: int
    utilization: float

    def as_dict(self) -> dict:
        return {"tiles": self.tiles, "useful_rows": self.useful_rows,
                "capacity": self.capacity, "utilization": self.utilization}


def _mask_host(mask, layout: BlockLayout) -> np.ndarray:
    m = mask.detach().to("cpu").numpy() if isinstance(mask, torch.Tensor) else np.asarray(mask)
    m = m.astype(np.int64, copy=False)
    if m.shape != (layout.n_q, layout.n_k):
        raise ValidationError(f"mask shape {m.shape} does not match layout "
                              f"{(layout.n_q, layout.n_k)}")
    if (m < 0).any() or (m > layout.levels).any():
        raise ValidationError(f"mask levels outside 0..{layout.levels}")
    return m


def build_schedule(mask, layout: BlockLayout, tile_len: int, merge: bool = True) -> TileSchedule:
    """Greedy in-order packing of the mask-selected pooled rows into tiles of ``tile_len`` rows
    (scheduler.py:71-126): blocks in ascending order, split across tiles when needed, tiles never
    span query blocks; ``merge=False`` starts every block in a fresh tile."""
    if tile_len < 1:
        raise ValidationError(f"tile_len must be >= 1, got {tile_len}")
    m = _mask_host(mask, layout)
    pooled = np.array([0] + [layout.pooled_len(h) for h in range(1, layout.levels + 1)])
    tiles = []
    for i in range(layout.n_q):
        js = np.nonzero(m[i])[0]
        if js.size == 0:
            continue
        lens = pooled[m[i, js]]
        if merge:  # one stream of rows; tile t covers [t*tile_len, (t+1)*tile_len)
            starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
        else:      # each block starts at a tile boundary
            tiles_per = -(-lens // tile_len)
            starts = np.concatenate([[0], np.cumsum(tiles_per)[:-1]]) * tile_len
        current, segs = None, []
        for j, h, s0, ln in zip(js.tolist(), m[i, js].tolist(), starts.tolist(), lens.tolist()):
            off = 0
            while off < ln:
                pos = s0 + off
                t = pos // tile_len
                take = min(ln - off, (t + 1) * tile_len - pos)
                if t != current:
                    if segs:
                        tiles.append(ExecutionTile(query_block=i, segments=tuple(segs)))
                    current, segs = t, []
                segs.append(Segment(kv_block=j, level=h, row_start=off, row_stop=off + take))
                off += take
        if segs:
            tiles.append(ExecutionTile(query_block=i, segments=tuple(segs)))
    return TileSchedule(tile_len=tile_len, tiles=tuple(tiles), layout=layout)


def utilization(schedule: TileSchedule) -> UtilizationStats:
    """Fill statistics of a schedule; 1.0 means every tile is full (scheduler.py:272-282)."""
    n_tiles = len(schedule.tiles)
    useful = sum(t.filled for t in schedule.tiles)
    capacity = n_tiles * schedule.tile_len
    return UtilizationStats(tiles=n_tiles, useful_rows=useful, capacity=capacity,
                            utilization=useful / capacity if capacity else 1.0)


def validate_schedule(schedule: TileSchedule, layout: BlockLayout) -> np.ndarray:
    """Reject schedules that would change attention semantics (scheduler.py:129-200) and return
    the (n_q, n_k) level map the schedule covers: within a query block, segments must cover
    whole selected blocks in strictly ascending block order without gaps, overlaps or level
    mixing."""
    if schedule.layout != layout:
        raise ValidationError("schedule layout does not match pyramid layout")
    if schedule.tile_len < 1:
        raise ValidationError("tile_len must be >= 1")
    mask = np.zeros((layout.n_q, layout.n_k), dtype=np.int64)
    last_qb, open_block, last_done = -1, None, -1

    def finish_open():
        nonlocal open_block, last_done
        if open_block is not None:
            j, h, nxt = open_block
            if nxt != layout.pooled_len(h):
                raise ValidationError(f"block {j} covered only to row {nxt} of "
                                      f"{layout.pooled_len(h)}")
            mask[last_qb, j] = h
            last_done, open_block = j, None

    for tile in schedule.tiles:
        if tile.query_block < last_qb or not 0 <= tile.query_block < layout.n_q:
            raise ValidationError("tiles out of query-block order")
        if tile.query_block != last_qb:
            finish_open()
            last_done, last_qb = -1, tile.query_block
        if not tile.segments:
            raise ValidationError("empty tile")
        if tile.filled > schedule.tile_len:
            raise ValidationError("tile overfull")
        for seg in tile.segments:
            if not 0 <= seg.kv_block < layout.n_k:
                raise ValidationError(f"segment block {seg.kv_block} out of range")
            if not 1 <= seg.level <= layout.levels:
                raise ValidationError(f"segment level {seg.level} out of range")
            limit = layout.pooled_len(seg.level)
            if not 0 <= seg.row_start < seg.row_stop <= limit:
                raise ValidationError(f"segment rows [{seg.row_start}, {seg.row_stop}) outside "
                                      f"0..{limit}")
            if open_block is not None and seg.kv_block == open_block[0]:
                j, h, nxt = open_block
                if seg.level != h:
                    raise ValidationError(f"block {j} mixes levels {h}/{seg.level}")
                if seg.row_start != nxt:
                    raise ValidationError(f"block {j} rows jump from {nxt} to {seg.row_start}")
                open_block = (j, h, seg.row_stop)
                continue
            finish_open()
            if seg.kv_block <= last_done:
                raise ValidationError(f"block {seg.kv_block} repeated or out of order")
            if seg.row_start != 0:
                raise ValidationError(f"block {seg.kv_block} does not start at row 0")
            open_block = (seg.kv_block, seg.level, seg.row_stop)
    finish_open()
    return mask


def execute_schedule(q, pyramid, schedule: TileSchedule, causal: bool = False):
    """Run a validated schedule on the GPU executor (scheduler.py:203-269). Returns the same
    AttentionOutput as psa_streaming on the schedule's mask."""
    from .attention import psa_streaming
    mask = validate_schedule(schedule, pyramid.layout)
    dev = pyramid.k_raw.device
    return psa_streaming(q, pyramid, torch.from_numpy(mask).to(dev), causal=causal)


def plan_utilization(plan, layout: BlockLayout, tile_rows: int = 128) -> UtilizationStats:
    """Fill of the tiles the sm_100a kernel executes for ``plan`` (MaskPlan): selected pooled
    rows over (tiles x 128); slot padding (e.g. 120-row blocks in 128-row slots) counts as
    unused."""
    counts = [int(c) for c in plan.level_counts.cpu().tolist()]
    useful = sum(c * layout.pooled_len(h) for h, c in enumerate(counts) if h >= 1)
    n_tiles = int(((plan.info[:, 1] + tile_rows - 1) // tile_rows).sum().item())
    capacity = n_tiles * tile_rows
    return UtilizationStats(tiles=n_tiles, useful_rows=useful, capacity=capacity,
                            utilization=useful / capacity if capacity else 1.0)

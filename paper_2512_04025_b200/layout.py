"""Block layout and the level/threshold configuration types of the PSA forward.

Host-side mirrors of the reference types with the same names, fields and validation:
  BlockLayout / make_layout           pkg/src/pyrattn/blocks.py:13-64
  SamplerConfig                       pkg/src/pyrattn/importance.py:22-38
  LevelThresholds / QuantileCutpoints / SimThresholds / PRESET_CUTPOINTS
                                      pkg/src/pyrattn/mask.py:20-97 (file lines 185-262)
Plus the GPU-kernel shape limits and the slot geometry the attention kernel uses.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ValidationError

TILE_ROWS = 128  # MMA tile (query rows and packed KV rows)


@dataclass(frozen=True)
class BlockLayout:
    """Partition of a length-N sequence into query blocks (b_q) and KV blocks (b_k).

    ``levels`` pyramid levels per KV block: level 1 is the raw block, level h has
    b_k / 2^(h-1) rows.
    """

    seq_len: int
    head_dim: int
    q_block: int
    k_block: int
    levels: int

    def __post_init__(self):
        if min(self.seq_len, self.head_dim, self.q_block, self.k_block) < 1:
            raise ValidationError("layout dimensions must be positive")
        if self.levels < 1:
            raise ValidationError(f"levels must be >= 1, got {self.levels}")
        for name, blk in (("q_block", self.q_block), ("k_block", self.k_block)):
            if self.seq_len % blk:
                raise ValidationError(f"seq_len {self.seq_len} not divisible by {name} {blk}")
        if self.k_block % (1 << (self.levels - 1)):
            raise ValidationError(
                f"k_block {self.k_block} not divisible by 2^{self.levels - 1}; "
                "the coarsest level would be empty")

    @property
    def n_q(self) -> int:
        return self.seq_len // self.q_block

    @property
    def n_k(self) -> int:
        return self.seq_len // self.k_block

    def pooled_len(self, level: int) -> int:
        if not 1 <= level <= self.levels:
            raise ValidationError(f"level {level} outside 1..{self.levels}")
        return self.k_block >> (level - 1)

    # ---- sm_100a kernel geometry (not part of the reference type)
    def slot_rows(self, level: int) -> int:
        """Rows a level-`level` segment occupies in a 128-row KV tile (power of two >= 8)."""
        rows = self.pooled_len(level)
        s = 8
        while s < rows:
            s <<= 1
        return s

    def check_gpu(self) -> None:
        if self.head_dim not in (64, 128):
            raise ValidationError(f"head_dim {self.head_dim} unsupported by the sm_100a kernels "
                                  "(64 or 128)")
        if self.q_block > TILE_ROWS or self.k_block > TILE_ROWS:
            raise ValidationError("q_block and k_block must be <= 128 for the sm_100a kernels")
        if self.n_k > 4096:
            raise ValidationError("n_k must be <= 4096")
        if self.levels > 8:
            raise ValidationError("levels must be <= 8 for the sm_100a kernels")


def make_layout(seq_len: int, head_dim: int, q_block: int, k_block: int,
                levels: int) -> BlockLayout:
    """Validated :class:`BlockLayout` (blocks.py:61-64)."""
    return BlockLayout(seq_len, head_dim, q_block, k_block, levels)


@dataclass(frozen=True)
class SamplerConfig:
    """Sampled-token counts and the seed of the sampled estimator."""

    s_q: int
    s_k: int
    seed: int

    def validate(self, layout: BlockLayout) -> None:
        if not 1 <= self.s_q <= layout.q_block:
            raise ValidationError(f"s_q={self.s_q} outside 1..{layout.q_block}")
        if not 1 <= self.s_k <= layout.k_block:
            raise ValidationError(f"s_k={self.s_k} outside 1..{layout.k_block}")


def _monotone_unit(vals, what: str) -> tuple:
    vals = tuple(float(t) for t in vals)
    if not vals:
        raise ValidationError(f"need at least one {what}")
    if vals[0] < 0.0 or vals[-1] > 1.0 or any(a > b for a, b in zip(vals, vals[1:])):
        raise ValidationError(f"{what}s must be non-decreasing within [0, 1], got {vals}")
    return vals


@dataclass(frozen=True)
class LevelThresholds:
    """Cumulative-importance budget per level (Alg. 2): non-decreasing in [0, 1]."""

    taus: tuple

    def __post_init__(self):
        object.__setattr__(self, "taus", _monotone_unit(self.taus, "threshold"))

    def __len__(self) -> int:
        return len(self.taus)


@dataclass(frozen=True)
class QuantileCutpoints:
    """Rank-fraction boundary per level: non-decreasing in [0, 1]."""

    points: tuple

    def __post_init__(self):
        object.__setattr__(self, "points", _monotone_unit(self.points, "cutpoint"))

    def __len__(self) -> int:
        return len(self.points)

    def counts(self, n_k: int) -> list:
        """Cumulative rank counts: floor(p*n_k + 0.5) clamped to n_k, running max
        (the reference's _fraction_counts, mask.py:161-164)."""
        out, run = [], 0
        for p in self.points:
            c = min(n_k, int(math.floor(p * n_k + 0.5)))
            run = max(run, c)
            out.append(run)
        return out


@dataclass(frozen=True)
class SimThresholds:
    """Minimum intra-block cosine similarity for levels 2..H, each in [-1, 1]."""

    taus: tuple

    def __post_init__(self):
        taus = tuple(float(t) for t in self.taus)
        if any(t < -1.0 or t > 1.0 for t in taus):
            raise ValidationError(f"similarity thresholds outside [-1, 1]: {taus}")
        object.__setattr__(self, "taus", taus)

    def __len__(self) -> int:
        return len(self.taus)


# Budget-matched presets (all 0.25x dense compute), same values as the reference table.
PRESET_CUTPOINTS = {
    "psa-1": QuantileCutpoints((0.25, 0.25, 0.25, 0.25)),
    "psa-2": QuantileCutpoints((0.0, 0.0, 1.0, 1.0)),
    "psa-3": QuantileCutpoints((0.15, 0.25, 0.45, 0.45)),
    "psa-4": QuantileCutpoints((0.10, 0.30, 0.50, 0.50)),
    "psa-5": QuantileCutpoints((0.10, 0.20, 0.60, 0.60)),
}

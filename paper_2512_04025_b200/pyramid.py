"""Pooled K/V pyramid (K1) and the similarity cap, on the GPU.

Drop-in for pkg/src/pyrattn/blocks.py:67-109 (PyramidKV, build_pyramid) and
pkg/src/pyrattn/mask.py:198-234 (level_cap_from_similarity). The pyramid lives in HBM as one
bf16 buffer per tensor holding levels 2..H back to back ([B, Hkv, N >> (h-1), d] each);
level 1 is the caller's K/V (never copied).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import as_bhnd, stream_handle
from .errors import ValidationError
from .layout import BlockLayout, SimThresholds


def pyramid_elems(bh: int, n: int, d: int, levels: int) -> int:
    return d * sum(bh * (n >> (h - 1)) for h in range(2, levels + 1))


@dataclass
class PyramidKV:
    """Per-level pooled keys/values of every (batch, kv-head).

    ``k(block, level)`` mirrors the reference accessor (blocks.py:78-83) and returns the
    (b_k / 2^(level-1), d) slice of KV block ``block`` for ``head``/``batch``.
    """

    layout: BlockLayout
    k_raw: torch.Tensor      # [B, Hkv, N, d] bf16
    v_raw: torch.Tensor
    k_pyr: torch.Tensor | None  # flat bf16 buffer, levels 2..H
    v_pyr: torch.Tensor | None

    @property
    def batch(self) -> int:
        return self.k_raw.shape[0]

    @property
    def heads(self) -> int:
        return self.k_raw.shape[1]

    def _level(self, buf, raw, level):
        lay = self.layout
        if not 1 <= level <= lay.levels:
            raise ValidationError(f"level {level} outside 1..{lay.levels}")
        if level == 1:
            return raw
        B, H, n, d = raw.shape
        off = pyramid_elems(B * H, n, d, level - 1)
        rows = n >> (level - 1)
        return buf[off: off + B * H * rows * d].view(B, H, rows, d)

    def level_k(self, level: int) -> torch.Tensor:
        return self._level(self.k_pyr, self.k_raw, level)

    def level_v(self, level: int) -> torch.Tensor:
        return self._level(self.v_pyr, self.v_raw, level)

    def k(self, block: int, level: int, head: int = 0, batch: int = 0) -> torch.Tensor:
        L = self.layout.pooled_len(level)
        return self.level_k(level)[batch, head, block * L:(block + 1) * L]

    def v(self, block: int, level: int, head: int = 0, batch: int = 0) -> torch.Tensor:
        L = self.layout.pooled_len(level)
        return self.level_v(level)[batch, head, block * L:(block + 1) * L]


def build_pyramid(k: torch.Tensor, v: torch.Tensor, layout: BlockLayout,
                  check_finite: bool = False, flag: torch.Tensor | None = None) -> PyramidKV:
    """Split K/V into KV blocks and pool each ``layout.levels`` deep (blocks.py:93-109).

    Levels are fp64 dyadic means of the bf16 inputs rounded once to bf16, i.e. exactly
    bf16(reference fp64 pyramid). ``check_finite`` makes the kernel flag NaN/Inf input and
    raises ValidationError like the reference's as_matrix (costs one host sync).
    """
    layout.check_gpu()
    k4, _ = as_bhnd(k, "K", layout.seq_len, layout.head_dim, stage=True)
    v4, _ = as_bhnd(v, "V", layout.seq_len, layout.head_dim, stage=True)
    if k4.shape != v4.shape:
        raise ValidationError(f"K/V shapes {tuple(k4.shape)}/{tuple(v4.shape)} differ")
    B, H, n, d = k4.shape
    dev = k4.device
    if layout.levels == 1:
        return PyramidKV(layout, k4, v4, None, None)
    total = pyramid_elems(B * H, n, d, layout.levels)
    kp = torch.empty(total, dtype=torch.bfloat16, device=dev)
    vp = torch.empty(total, dtype=torch.bfloat16, device=dev)
    # ``flag`` (device int32 [1]): set when K or V holds NaN/Inf, without a host sync
    if check_finite and flag is None:
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    rc = lib.psa_pyramid_build(k4.data_ptr(), v4.data_ptr(), B * H, n, d, layout.k_block,
                               layout.levels, kp.data_ptr(), vp.data_ptr(), _lib.ptr(flag),
                               stream_handle(dev))
    _lib.check(rc, "psa_pyramid_build")
    if check_finite and int(flag.item()):
        raise ValidationError("K or V contains NaN or Inf entries")
    return PyramidKV(layout, k4, v4, kp, vp)


def build_pyramid_gather(k4: torch.Tensor, v4: torch.Tensor, layout: BlockLayout,
                         index: torch.Tensor) -> PyramidKV:
    """Pyramid of the token-permuted K/V (pipeline.py:257-263 then blocks.py:93-109) in one pass:
    the permutation is a gather in the pyramid kernel's loads (psa_pyramid_build_gather). The
    returned PyramidKV's level 1 (``k_raw``/``v_raw``) is the permuted K/V."""
    layout.check_gpu()
    if k4.shape != v4.shape or k4.dim() != 4 or not (k4.is_contiguous() and v4.is_contiguous()):
        raise ValidationError("K/V must be contiguous [B, H, N, d] tensors of one shape")
    B, H, n, d = k4.shape
    if index.numel() != n or index.dtype != torch.int64 or index.device != k4.device:
        raise ValidationError(f"permutation must be a device int64 tensor of {n} entries")
    k1, v1 = torch.empty_like(k4), torch.empty_like(v4)
    kp = vp = None
    if layout.levels > 1:
        total = pyramid_elems(B * H, n, d, layout.levels)
        kp = torch.empty(total, dtype=torch.bfloat16, device=k4.device)
        vp = torch.empty(total, dtype=torch.bfloat16, device=k4.device)
    rc = _lib.load().psa_pyramid_build_gather(
        k4.data_ptr(), v4.data_ptr(), B * H, n, d, layout.k_block, layout.levels, index.data_ptr(),
        k1.data_ptr(), v1.data_ptr(), _lib.ptr(kp), _lib.ptr(vp), None, stream_handle(k4.device))
    _lib.check(rc, "psa_pyramid_build_gather")
    return PyramidKV(layout, k1, v1, kp, vp)


def similarity_caps(k4: torch.Tensor, layout: BlockLayout, sim: SimThresholds) -> torch.Tensor:
    """int8 caps [B, Hkv, n_k] from raw keys (device)."""
    if len(sim) != layout.levels - 1:
        raise ValidationError(f"need {layout.levels - 1} similarity thresholds for "
                              f"{layout.levels} levels, got {len(sim)}")
    B, H, n, d = k4.shape
    caps = torch.empty(B, H, layout.n_k, dtype=torch.int8, device=k4.device)
    taus = _lib.host_doubles(sim.taus)
    rc = _lib.load().psa_similarity_caps(k4.data_ptr(), B * H, n, d, layout.k_block,
                                         layout.levels, taus, caps.data_ptr(),
                                         stream_handle(k4.device))
    _lib.check(rc, "psa_similarity_caps")
    return caps


def level_cap_from_similarity(source, sim_thresholds: SimThresholds,
                              layout: BlockLayout | None = None) -> torch.Tensor:
    """Per-KV-block maximum admissible level (mask.py:198-234), int64.

    ``source`` is a PyramidKV or a raw key tensor with an explicit layout. Returns (n_k,) for a
    single head input, else [..., n_k] following the input's leading dims.
    """
    if isinstance(source, PyramidKV):
        layout = source.layout
        k4 = source.k_raw
        lead = tuple(k4.shape[:2]) if k4.shape[:2] != (1, 1) else ()
    else:
        if layout is None:
            raise ValidationError("raw key input requires an explicit layout")
        k4, lead = as_bhnd(source, "K", layout.seq_len, layout.head_dim, stage=True)
    layout.check_gpu()
    caps = similarity_caps(k4, layout, sim_thresholds)
    return caps.to(torch.int64).reshape(lead + (layout.n_k,))

"""Multi-level block-sparse attention (K4) and the dense yardsticks.

Drop-ins for pkg/src/pyrattn/attention.py:
  AttentionOutput :25-36, level_bias :39-44, full_attention :47-63,
  psa_streaming :171-218, causal_full_attention :221-241.
All of them run the tcgen05/TMEM kernel in libpsa (psa_attn_fwd); the dense variants are the
same kernel on an all-level-1 plan.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import as_bhnd, check_finite, restore, stream_handle, to_device
from .errors import ValidationError
from .layout import BlockLayout, make_layout
from .mask import MaskPlan, causal_premask, plan_from_mask
from .pyramid import PyramidKV, build_pyramid

LN2 = math.log(2.0)


@dataclass
class AttentionOutput:
    """Attention result: ``out`` (bf16), natural-log row normalisers (-inf for rows with no
    key; such rows are zero in ``out``) and the number of such rows."""

    out: torch.Tensor
    row_log_normalizers: torch.Tensor
    skipped_rows: int = 0


def level_bias(level: int, max_level: int | None = None) -> float:
    """Additive logit bias (h-1)*ln 2 of pooling level h."""
    if level < 1 or (max_level is not None and level > max_level):
        hi = max_level if max_level is not None else "inf"
        raise ValidationError(f"level {level} outside 1..{hi}")
    return (level - 1) * LN2


def attention_forward(q4: torch.Tensor, pyr: PyramidKV, plan: MaskPlan, causal: bool,
                      out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                      skipped: torch.Tensor | None = None, out_rows: torch.Tensor | None = None,
                      qblocks: torch.Tensor | None = None):
    """Launch psa_attn_fwd on device tensors; returns (out, lse, skipped-counter). ``out_rows``
    (device int64 [n]): store O/lse row i of every head at row out_rows[i] (fused unpermute).
    ``qblocks`` (device int32): only these query blocks (the plan's rows); O/lse are then
    compact, [B, Hq, len(qblocks) * b_q, ...]."""
    lay = pyr.layout
    B, Hq, n, d = q4.shape
    Hkv = pyr.k_raw.shape[1]
    if pyr.k_raw.shape[0] != B or Hq % Hkv:
        raise ValidationError(f"Q heads {Hq} / batch {B} incompatible with K/V "
                              f"{tuple(pyr.k_raw.shape)}")
    dev = q4.device
    if qblocks is not None:
        if out_rows is not None:
            raise ValidationError("the row scatter and query-block subsets are exclusive")
        rows = qblocks.numel() * lay.q_block
        out = torch.empty(B, Hq, rows, d, dtype=q4.dtype, device=dev) if out is None else out
        lse = torch.empty(B, Hq, rows, dtype=torch.float32, device=dev) if lse is None else lse
        if skipped is None:
            skipped = torch.zeros(1, dtype=torch.int32, device=dev)
        rc = _lib.load().psa_attn_fwd_rows(
            q4.data_ptr(), pyr.k_raw.data_ptr(), pyr.v_raw.data_ptr(), _lib.ptr(pyr.k_pyr),
            _lib.ptr(pyr.v_pyr), B, Hq, Hkv, n, d, lay.q_block, lay.k_block, lay.levels,
            plan.csr.data_ptr(), plan.info.data_ptr(), int(causal), qblocks.data_ptr(),
            qblocks.numel(), out.data_ptr(), lse.data_ptr(), skipped.data_ptr(),
            stream_handle(dev))
        _lib.check(rc, "psa_attn_fwd")
        return out, lse, skipped
    out = torch.empty_like(q4) if out is None else out
    lse = torch.empty(B, Hq, n, dtype=torch.float32, device=dev) if lse is None else lse
    if skipped is None:
        skipped = torch.zeros(1, dtype=torch.int32, device=dev)
    if out_rows is not None and (out_rows.numel() != n or out_rows.dtype != torch.int64
                                 or out_rows.device != dev):
        raise ValidationError(f"out_rows must be a device int64 tensor of {n} entries")
    rc = _lib.load().psa_attn_fwd_scatter(
        q4.data_ptr(), pyr.k_raw.data_ptr(), pyr.v_raw.data_ptr(), _lib.ptr(pyr.k_pyr),
        _lib.ptr(pyr.v_pyr), B, Hq, Hkv, n, d, lay.q_block, lay.k_block, lay.levels,
        plan.csr.data_ptr(), plan.info.data_ptr(), int(causal), out.data_ptr(), lse.data_ptr(),
        skipped.data_ptr(), _lib.ptr(out_rows), stream_handle(dev))
    _lib.check(rc, "psa_attn_fwd")
    return out, lse, skipped


def attention_backward(q4: torch.Tensor, pyr: PyramidKV, plan: MaskPlan, causal: bool,
                       out: torch.Tensor, lse: torch.Tensor, dout: torch.Tensor):
    """Gradients (dq, dk, dv) of attention_forward for the fixed mask ``plan`` (psa_attn_bwd):
    dk/dv are w.r.t. the raw K/V of ``pyr`` (pooled levels differentiated through their means).
    Limit (include/psa.h): about 5.6K (query head, query block) entries per KV head, i.e.
    (Hq / Hkv) * n_q; larger shapes raise the library's "too many query blocks per KV head"."""
    lay = pyr.layout
    B, Hq, n, d = q4.shape
    Hkv = pyr.k_raw.shape[1]
    dev = q4.device
    dout = dout.to(torch.bfloat16).contiguous()
    if dout.shape != q4.shape or out.shape != q4.shape or lse.shape != q4.shape[:-1]:
        raise ValidationError("out / lse / dout shapes do not match q")
    dq = torch.empty_like(q4)
    dk = torch.empty_like(pyr.k_raw)
    dv = torch.empty_like(pyr.v_raw)
    lib = _lib.load()
    ws = torch.empty(lib.psa_attn_bwd_workspace_bytes(B, Hq, Hkv, n, d), dtype=torch.uint8, device=dev)
    rc = lib.psa_attn_bwd(
        q4.data_ptr(), pyr.k_raw.data_ptr(), pyr.v_raw.data_ptr(), _lib.ptr(pyr.k_pyr),
        _lib.ptr(pyr.v_pyr), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), B, Hq, Hkv, n, d,
        lay.q_block, lay.k_block, lay.levels, plan.csr.data_ptr(), plan.info.data_ptr(),
        plan.level_map.data_ptr(), int(causal), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
        ws.data_ptr(), stream_handle(dev))
    _lib.check(rc, "psa_attn_bwd")
    return dq, dk, dv


def psa_streaming(q, pyramid: PyramidKV, mask, causal: bool = False) -> AttentionOutput:
    """Multi-level attention over the mask-selected (block, level) pairs (attention.py:171-218).

    ``mask`` has shape (n_q, n_k) for single-head input or [..., n_q, n_k] following q's leading
    dims. Output ``out`` is bf16; ``row_log_normalizers`` fp32.
    """
    lay = pyramid.layout
    lay.check_gpu()
    q4, lead = as_bhnd(q, "Q", lay.seq_len, lay.head_dim, stage=True)
    check_finite("Q", q4)
    mask = to_device(mask, "mask")
    B, Hq = q4.shape[:2]
    if tuple(mask.shape[-2:]) != (lay.n_q, lay.n_k) or mask.numel() != B * Hq * lay.n_q * lay.n_k:
        raise ValidationError(f"mask shape {tuple(mask.shape)} does not match layout "
                              f"{(lay.n_q, lay.n_k)} for {B}x{Hq} heads")
    plan = plan_from_mask(mask, lay, causal, B, Hq)
    out, lse, skipped = attention_forward(q4, pyramid, plan, causal)
    return AttentionOutput(out=restore(out, lead), row_log_normalizers=lse.reshape(lead + (lay.seq_len,)),
                           skipped_rows=int(skipped.item()))


def psa_reference(q, pyramid: PyramidKV, mask, causal: bool = False) -> AttentionOutput:
    """Materialized multi-level attention (attention.py:120-168). In the reference this is the
    ground truth for the streaming pass; on the GPU both are the same sm_100a kernel (the
    per-block softmax is computed exactly once either way), so this returns psa_streaming."""
    return psa_streaming(q, pyramid, mask, causal=causal)


def _dense_layout(n: int, d: int) -> BlockLayout:
    for b in (128, 120, 112, 96, 64, 32, 16, 8):
        if n % b == 0:
            return make_layout(n, d, b, b, 1)
    raise ValidationError(f"seq_len {n} has no block size <= 128 that is a multiple of 8")


def _dense(q, k, v, causal: bool) -> AttentionOutput:
    q4, lead = as_bhnd(q, "Q", stage=True)
    k4, _ = as_bhnd(k, "K", q4.shape[2], q4.shape[3], stage=True)
    v4, _ = as_bhnd(v, "V", q4.shape[2], q4.shape[3], stage=True)
    check_finite("Q / K / V", q4, k4, v4)
    if k4.shape != v4.shape:
        raise ValidationError(f"incompatible shapes K{tuple(k4.shape)} V{tuple(v4.shape)}")
    lay = _dense_layout(q4.shape[2], q4.shape[3])
    lay.check_gpu()
    B, Hq = q4.shape[:2]
    m = torch.ones(B, Hq, lay.n_q, lay.n_k, dtype=torch.int64, device=q4.device)
    if causal:
        m = causal_premask(m, lay)
    pyr = build_pyramid(k4, v4, lay)
    plan = plan_from_mask(m, lay, causal, B, Hq)
    out, lse, skipped = attention_forward(q4, pyr, plan, causal)
    return AttentionOutput(out=restore(out, lead), row_log_normalizers=lse.reshape(lead + (lay.seq_len,)),
                           skipped_rows=int(skipped.item()))


def full_attention(q, k, v) -> AttentionOutput:
    """Dense softmax(Q K^T / sqrt(d)) V (attention.py:47-63) with the same kernel."""
    return _dense(q, k, v, causal=False)


def causal_full_attention(q, k, v) -> AttentionOutput:
    """Dense attention with a token-level causal mask (attention.py:221-241)."""
    return _dense(q, k, v, causal=True)

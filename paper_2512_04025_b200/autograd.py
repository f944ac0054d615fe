"""Differentiable PSA forward: torch.autograd over the sm_100a kernels.

The forward is the fused pipeline (pyramid -> importance -> level map -> attention); the mask is
a discrete decision and carries no gradient, exactly like a block-sparse attention mask in
training. The backward is ``psa_attn_bwd`` (psa_backward.cu): dQ, and dK/dV w.r.t. the raw keys
and values through the pooled levels. The reference has no backward; the test
oracle is the autograd of the forward's definition in fp64 (tests/test_gpu_backward.py).
"""

from __future__ import annotations

import torch

from ._tensors import as_bhnd, restore
from .errors import ValidationError


class _PSAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q4, k4, v4, cfg):
        from .pipeline import psa_forward_4d
        res = psa_forward_4d(q4, k4, v4, cfg)
        # K/V ride in the saved tensors too (the pyramid's level 1 is the caller's K/V), so an
        # in-place edit between forward and backward trips autograd's version check
        ctx.save_for_backward(q4, k4, v4, res.out, res.lse)
        ctx.pyr, ctx.plan, ctx.causal = res.pyramid, res.plan, cfg.causal
        ctx.mark_non_differentiable(res.lse)
        return res.out, res.lse

    @staticmethod
    def backward(ctx, dout, _dlse):
        from .attention import attention_backward
        q4, _k4, _v4, out, lse = ctx.saved_tensors
        dq, dk, dv = attention_backward(q4, ctx.pyr, ctx.plan, ctx.causal, out, lse, dout)
        return dq, dk, dv, None


def psa_attention_differentiable(q, k, v, cfg=None, **overrides):
    """``psa_attention`` returning (out, lse) that supports ``backward()`` w.r.t. q, k and v
    (CUDA bf16 tensors shaped (n, d), (H, n, d) or (B, H, n, d)). The token permutation
    (``grid``) is not supported on this path yet."""
    from .pipeline import resolve_config
    q4, lead = as_bhnd(q, "Q")
    k4, _ = as_bhnd(k, "K")
    v4, _ = as_bhnd(v, "V")
    cfg = resolve_config(cfg, q4.shape[2], q4.shape[3], overrides)
    if cfg.grid is not None:
        raise ValidationError("the differentiable path does not support grid permutations yet")
    out, lse = _PSAFunction.apply(q4, k4, v4, cfg)
    return restore(out, lead), lse.reshape(lead + (q4.shape[2],))

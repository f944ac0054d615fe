"""Tensor plumbing shared by the drop-in entry points: shape normalisation to [B, H, N, d],
device/dtype checks (no CPU fallback), and the current CUDA stream handle."""

from __future__ import annotations

import torch

from .errors import ValidationError


def require_cuda(x: torch.Tensor, name: str) -> None:
    if not isinstance(x, torch.Tensor):
        raise ValidationError(f"{name} must be a torch.Tensor on a CUDA device")
    if not x.is_cuda:
        raise ValidationError(f"{name} must live on a CUDA device: the sm_100a kernels are the "
                              "only implementation (no CPU fallback)")


def to_device(x, name: str) -> torch.Tensor:
    """Array-likes and host tensors (the reference accepts anything as_matrix converts,
    pkg/src/pyrattn/linalg.py:15-24) are staged onto the current CUDA device; CUDA tensors pass
    through. Without a CUDA device this raises: there is no CPU implementation."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x
    if not torch.cuda.is_available():
        raise ValidationError(f"{name} must live on a CUDA device: the sm_100a kernels are the only "
                              "implementation (no CPU fallback)")
    if not isinstance(x, torch.Tensor):
        import numpy as np
        try:
            arr = np.asarray(x)
        except Exception as exc:  # noqa: BLE001
            raise ValidationError(f"{name} is not array-like: {exc}") from exc
        if arr.dtype == object or not (np.issubdtype(arr.dtype, np.floating)
                                       or np.issubdtype(arr.dtype, np.integer)
                                       or arr.dtype == np.bool_):
            raise ValidationError(f"{name} must be a numeric array, got dtype {arr.dtype}")
        x = torch.from_numpy(np.ascontiguousarray(arr))
    return x.to(torch.device("cuda", torch.cuda.current_device()))


def check_finite(name: str, *xs: torch.Tensor) -> None:
    """ValidationError on NaN / Inf entries, as the reference's as_matrix (linalg.py:15-24)."""
    for x in xs:
        if not bool(torch.isfinite(x).all()):
            raise ValidationError(f"{name} contains NaN or Inf entries")


def as_bhnd(x, name: str, n: int | None = None, d: int | None = None, stage: bool = False):
    """Return (x as contiguous bf16 [B, H, N, d], original leading shape). ``stage``: accept
    array-likes / host tensors and copy them to the current CUDA device."""
    if stage:
        x = to_device(x, name)
    require_cuda(x, name)
    if x.ndim not in (2, 3, 4):
        raise ValidationError(f"{name} must be (n, d), (heads, n, d) or (batch, heads, n, d), "
                              f"got shape {tuple(x.shape)}")
    lead = tuple(x.shape[:-2])
    if x.numel() == 0:
        raise ValidationError(f"{name} must be non-empty, got shape {tuple(x.shape)}")
    if not x.is_floating_point():
        raise ValidationError(f"{name} must be a floating-point tensor")
    x4 = x.reshape((1,) * (4 - x.ndim) + tuple(x.shape))
    if n is not None and x4.shape[2] != n:
        raise ValidationError(f"{name} has {x4.shape[2]} rows, layout expects {n}")
    if d is not None and x4.shape[3] != d:
        raise ValidationError(f"{name} head_dim {x4.shape[3]} does not match layout {d}")
    if x4.dtype != torch.bfloat16:
        x4 = x4.to(torch.bfloat16)
    return x4.contiguous(), lead


def restore(x4: torch.Tensor, lead: tuple) -> torch.Tensor:
    return x4.reshape(lead + tuple(x4.shape[2:]))


def stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream

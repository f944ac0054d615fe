"""Space-filling-curve token permutations on the GPU path.

Drop-ins for pkg/src/pyrattn/permute.py: Permutation :21-38, hilbert_order :97-128,
apply_permutation :131-137, invert_permutation :140-141.

The curve itself is index bookkeeping that depends only on the grid (like the importance sample
tables): it is generated once per grid on the host -- the generalized Hilbert ("gilbert") walk of
permute.py:46-90, written here as an explicit-stack traversal that emits cells in the same order
as the reference's recursive generator -- and cached on each device. Applying a permutation to
Q/K/V/O is a row gather in libpsa (psa_gather_rows), HBM-bound.
"""

from __future__ import annotations

import functools

import numpy as np
import torch

from . import _lib
from ._tensors import require_cuda, stream_handle
from .errors import ValidationError


def _sgn(v: int) -> int:
    return (v > 0) - (v < 0)


def _gilbert_cells(x0: int, y0: int, ax0: int, ay0: int, bx0: int, by0: int) -> list:
    """Cells of the generalized Hilbert walk over the rectangle spanned by (ax, ay), (bx, by)
    from (x, y) (permute.py:46-90), in walk order, without recursion."""
    out = []
    stack = [(x0, y0, ax0, ay0, bx0, by0)]
    while stack:
        x, y, ax, ay, bx, by = stack.pop()
        w, h = abs(ax + ay), abs(bx + by)
        dax, day, dbx, dby = _sgn(ax), _sgn(ay), _sgn(bx), _sgn(by)
        if h == 1:
            out.extend((x + t * dax, y + t * day) for t in range(w))
            continue
        if w == 1:
            out.extend((x + t * dbx, y + t * dby) for t in range(h))
            continue
        ax2, ay2, bx2, by2 = ax // 2, ay // 2, bx // 2, by // 2
        w2, h2 = abs(ax2 + ay2), abs(bx2 + by2)
        if 2 * w > 3 * h:
            if (w2 % 2) and w > 2:
                ax2, ay2 = ax2 + dax, ay2 + day
            parts = [(x, y, ax2, ay2, bx, by),
                     (x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by)]
        else:
            if (h2 % 2) and h > 2:
                bx2, by2 = bx2 + dbx, by2 + dby
            parts = [(x, y, bx2, by2, ax2, ay2),
                     (x + bx2, y + by2, ax, ay, bx - bx2, by - by2),
                     (x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby),
                      -bx2, -by2, -(ax - ax2), -(ay - ay2))]
        stack.extend(reversed(parts))  # first part on top: same order as the recursion
    return out


def _walk2d(n0: int, n1: int) -> list:
    if n0 >= n1:
        return _gilbert_cells(0, 0, n0, 0, 0, n1)
    return [(x, y) for (y, x) in _gilbert_cells(0, 0, n1, 0, 0, n0)]


@functools.lru_cache(maxsize=32)
def _order_host(grid: tuple) -> np.ndarray:
    if len(grid) == 2:
        n0, n1 = grid
        flat = [x * n1 + y for (x, y) in _walk2d(n0, n1)]
    else:
        n0, n1, n2 = grid
        plane = _walk2d(n1, n2)
        flat = []
        for s in range(n0):
            if s:
                plane = plane[::-1]  # serpentine: re-enter where the last plane ended
            flat.extend(s * n1 * n2 + x * n2 + y for (x, y) in plane)
    return np.asarray(flat, dtype=np.int64)


class Permutation:
    """A bijection on token indices with its inverse (permute.py:21-38). ``order``/``inverse``
    are int64 host tensors; ``on(device)`` returns cached device copies."""

    def __init__(self, order):
        o = torch.as_tensor(np.asarray(order.cpu() if isinstance(order, torch.Tensor) else order),
                            dtype=torch.int64).reshape(-1).contiguous()
        n = o.numel()
        if not torch.equal(torch.sort(o).values, torch.arange(n, dtype=torch.int64)):
            raise ValidationError("order is not a bijection on 0..n-1")
        inv = torch.empty_like(o)
        inv[o] = torch.arange(n, dtype=torch.int64)
        self.order, self.inverse = o, inv
        self._dev = {}

    def __len__(self) -> int:
        return self.order.numel()

    def on(self, device) -> tuple:
        key = str(device)
        if key not in self._dev:
            self._dev[key] = (self.order.to(device), self.inverse.to(device))
        return self._dev[key]


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


@functools.lru_cache(maxsize=32)
def _hilbert_cached(grid: tuple) -> Permutation:
    return Permutation(_order_host(grid))


def hilbert_order(grid) -> Permutation:
    """Curve order for a 2D (power-of-two axes) or 3D (serpentine of 2D walks) grid over
    row-major tokens: entry i is the flat index of the i-th cell on the curve
    (permute.py:97-128)."""
    grid = tuple(int(g) for g in grid)
    if len(grid) not in (2, 3):
        raise ValidationError(f"grid must have 2 or 3 axes, got {len(grid)}")
    if min(grid) < 1:
        raise ValidationError("grid axes must be positive")
    if len(grid) == 2 and not (_is_pow2(grid[0]) and _is_pow2(grid[1])):
        raise ValidationError(f"2D grid axes must be powers of two, got {grid[0]}x{grid[1]}")
    return _hilbert_cached(grid)


def gather_rows(x4: torch.Tensor, index: torch.Tensor, out: torch.Tensor | None = None):
    """out[b, h, i] = x4[b, h, index[i]] for a contiguous bf16 [B, H, N, d] device tensor."""
    B, H, n, d = x4.shape
    if index.numel() != n:
        raise ValidationError(f"permutation covers {index.numel()} rows but sequence has {n}")
    out = torch.empty_like(x4) if out is None else out
    rc = _lib.load().psa_gather_rows(x4.data_ptr(), B * H, n, d * x4.element_size(),
                                     index.data_ptr(), out.data_ptr(), stream_handle(x4.device))
    _lib.check(rc, "psa_gather_rows")
    return out


def apply_permutation(x: torch.Tensor, p: Permutation) -> torch.Tensor:
    """Reorder the token rows of ``x`` ((n, d), (H, n, d) or (B, H, n, d) CUDA tensor) so that
    output row i is input row order[i] (permute.py:131-137)."""
    require_cuda(x, "sequence")
    if x.ndim < 2 or x.shape[-2] != len(p):
        raise ValidationError(f"permutation covers {len(p)} rows but sequence has "
                              f"{x.shape[-2] if x.ndim >= 2 else 0}")
    x4 = x.reshape((1,) * (4 - x.ndim) + tuple(x.shape)).contiguous()
    order, _ = p.on(x.device)
    return gather_rows(x4, order).reshape(x.shape)


def invert_permutation(p: Permutation) -> Permutation:
    """permute.py:140-141."""
    return Permutation(p.inverse.clone())

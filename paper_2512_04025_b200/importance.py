"""Block-importance estimation (K2) on the GPU.

Drop-ins for importance_sampled (pkg/src/pyrattn/importance.py:52-85), antidiagonal_selection
(:88-94) and importance_antidiagonal (:97-132). The sampled row
indices come from the same single seeded numpy generator in the same order as the reference
(importance.py:68-76: every query block ascending, then every KV block ascending); they
depend only on (seed, layout, s_q, s_k), are shared by all heads, and are cached on the
device. All tensor arithmetic (fp64 logits, softmax statistics, block max) runs in libpsa.
"""

from __future__ import annotations

import functools

import numpy as np
import torch

from . import _lib
from ._tensors import as_bhnd, check_finite, stream_handle
from .errors import ValidationError
from .layout import BlockLayout, SamplerConfig


@functools.lru_cache(maxsize=64)
def _sample_tables_host(seed: int, n_q: int, b_q: int, s_q: int, n_k: int, b_k: int, s_k: int):
    rng = np.random.default_rng(seed)
    q_rows = np.concatenate([i * b_q + rng.permutation(b_q)[:s_q] for i in range(n_q)])
    k_rows = np.concatenate([j * b_k + rng.permutation(b_k)[:s_k] for j in range(n_k)])
    return q_rows.astype(np.int32), k_rows.astype(np.int32)


_device_tables: dict = {}


def sample_tables(layout: BlockLayout, cfg: SamplerConfig, device) -> tuple:
    """(q_rows, k_rows) int32 device tensors of sampled row indices inside a head."""
    key = (cfg.seed, layout.n_q, layout.q_block, cfg.s_q, layout.n_k, layout.k_block, cfg.s_k,
           str(device))
    hit = _device_tables.get(key)
    if hit is None:
        qr, kr = _sample_tables_host(*key[:-1])
        hit = (torch.from_numpy(qr).to(device), torch.from_numpy(kr).to(device))
        _device_tables[key] = hit
    return hit


def _flags(fp64_only: bool) -> int:
    return _lib.PSA_IMP_FP64_ONLY if fp64_only else 0


def query_blocks(qblocks, layout: BlockLayout, device) -> torch.Tensor | None:
    """Validate a query-block subset (the (b, h, q-block set) work units of parallel.py) and
    return it as a device int32 tensor, or None for every block."""
    if qblocks is None:
        return None
    if getattr(qblocks, "_psa_n_q", None) == layout.n_q and qblocks.device == torch.device(device):
        return qblocks  # validated already (no host round trip: capturable in a CUDA graph)
    blk = torch.as_tensor(qblocks, dtype=torch.int64).reshape(-1).cpu()
    if blk.numel() == 0 or int(blk.min()) < 0 or int(blk.max()) >= layout.n_q:
        raise ValidationError(f"query blocks must be a non-empty subset of 0..{layout.n_q - 1}")
    if torch.unique(blk).numel() != blk.numel():
        raise ValidationError("query blocks must be distinct")
    out = blk.to(torch.int32).to(device)
    out._psa_n_q = layout.n_q
    return out


def importance_scores(q4: torch.Tensor, k4: torch.Tensor, layout: BlockLayout,
                      cfg: SamplerConfig, reducer: str = "max",
                      fp64_only: bool = False, qblocks=None) -> torch.Tensor:
    """fp64 scores [B, Hq, n_q, n_k] from bf16 [B, H, N, d] device tensors.

    Logits are exact (int8-sliced tensor cores, psa_xlogits.cu); ``fp64_only`` forces the fp64
    DMMA kernel instead (same values; used to cross-check the two paths). ``qblocks``: only
    these query blocks (rows of the result, in that order; the reference's sample rows of those
    blocks, so each row equals the full call's)."""
    if reducer not in ("max", "mean"):
        raise ValidationError(f"reducer must be 'max' or 'mean', got {reducer!r}")
    cfg.validate(layout)
    if cfg.s_k > 64:
        raise ValidationError("s_k > 64 is not supported by the sm_100a importance kernel")
    B, Hq, n, d = q4.shape
    Hkv = k4.shape[1]
    if Hq % Hkv:
        raise ValidationError(f"query heads {Hq} not a multiple of kv heads {Hkv}")
    dev = q4.device
    q_rows, k_rows = sample_tables(layout, cfg, dev)
    blk = query_blocks(qblocks, layout, dev)
    n_sel = layout.n_q
    if blk is not None:  # the table rows of the listed blocks, block-major
        n_sel = blk.numel()
        q_rows = q_rows.view(layout.n_q, cfg.s_q)[blk.long()].reshape(-1).contiguous()
    lib = _lib.load()
    ws_bytes = lib.psa_importance_workspace_bytes(B * Hq, B * Hkv, n_sel, cfg.s_q,
                                                  layout.n_k, cfg.s_k)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    scores = torch.empty(B, Hq, n_sel, layout.n_k, dtype=torch.float64, device=dev)
    rc = lib.psa_importance_sampled_rows(q4.data_ptr(), k4.data_ptr(), B, Hq, Hkv, n, d,
                                         layout.q_block, layout.k_block, q_rows.data_ptr(),
                                         k_rows.data_ptr(), cfg.s_q, cfg.s_k,
                                         0 if reducer == "max" else 1, _flags(fp64_only), n_sel,
                                         scores.data_ptr(), ws.data_ptr(), stream_handle(dev))
    _lib.check(rc, "psa_importance_sampled")
    return scores


def importance_sampled(q, k, layout: BlockLayout, cfg: SamplerConfig,
                       reducer: str = "max") -> torch.Tensor:
    """Sampled-token importance scores (importance.py:52-85), float64.

    Shape (n_q, n_k) for (n, d) inputs, else [..., n_q, n_k] following q's leading dims.
    """
    layout.check_gpu()
    q4, lead = as_bhnd(q, "Q", layout.seq_len, layout.head_dim, stage=True)
    k4, _ = as_bhnd(k, "K", layout.seq_len, layout.head_dim, stage=True)
    check_finite("Q / K", q4, k4)
    s = importance_scores(q4, k4, layout, cfg, reducer)
    return s.reshape(lead + (layout.n_q, layout.n_k))


def antidiagonal_selection(b_q: int, b_k: int, stride: int) -> torch.Tensor:
    """Boolean (b_q, b_k) mask of the strided antidiagonal positions (importance.py:88-94).
    A host-side layout helper (no tensor data), as in the reference."""
    if stride < 1 or b_k % stride:
        raise ValidationError(f"stride {stride} must divide k_block {b_k}")
    p = torch.arange(b_q)[:, None]
    c = torch.arange(b_k)[None, :]
    return (p + c) % stride == 0


def antidiagonal_scores(q4: torch.Tensor, k4: torch.Tensor, layout: BlockLayout,
                        stride: int, fp64_only: bool = False, qblocks=None) -> torch.Tensor:
    """fp64 antidiagonal scores [B, Hq, n_q, n_k] from bf16 [B, H, N, d] device tensors
    (``qblocks``: only these query blocks, rows in that order)."""
    if stride is None or int(stride) < 1 or layout.k_block % int(stride):
        raise ValidationError(f"stride {stride} must divide k_block {layout.k_block}")
    stride = int(stride)
    if layout.k_block // stride > 64:
        raise ValidationError("k_block / stride > 64 is not supported by the sm_100a "
                              "antidiagonal kernel")
    B, Hq, n, d = q4.shape
    Hkv = k4.shape[1]
    if Hq % Hkv:
        raise ValidationError(f"query heads {Hq} not a multiple of kv heads {Hkv}")
    dev = q4.device
    blk = query_blocks(qblocks, layout, dev)
    n_sel = layout.n_q if blk is None else blk.numel()
    lib = _lib.load()
    ws = torch.empty(lib.psa_antidiag_workspace_bytes_rows(B * Hq, B * Hkv, n, layout.q_block,
                                                           layout.k_block, stride, n_sel),
                     dtype=torch.uint8, device=dev)
    scores = torch.empty(B, Hq, n_sel, layout.n_k, dtype=torch.float64, device=dev)
    rc = lib.psa_importance_antidiagonal_rows(q4.data_ptr(), k4.data_ptr(), B, Hq, Hkv, n, d,
                                              layout.q_block, layout.k_block, stride,
                                              _flags(fp64_only), _lib.ptr(blk), n_sel,
                                              scores.data_ptr(), ws.data_ptr(),
                                              stream_handle(dev))
    _lib.check(rc, "psa_importance_antidiagonal")
    return scores


def importance_antidiagonal(q, k, layout: BlockLayout, stride: int) -> torch.Tensor:
    """Antidiagonal-probe importance scores (importance.py:97-132), float64.

    Shape (n_q, n_k) for (n, d) inputs, else [..., n_q, n_k] following q's leading dims.
    """
    layout.check_gpu()
    q4, lead = as_bhnd(q, "Q", layout.seq_len, layout.head_dim, stage=True)
    k4, _ = as_bhnd(k, "K", layout.seq_len, layout.head_dim, stage=True)
    check_finite("Q / K", q4, k4)
    s = antidiagonal_scores(q4, k4, layout, stride)
    return s.reshape(lead + (layout.n_q, layout.n_k))

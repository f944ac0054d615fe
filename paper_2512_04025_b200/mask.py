"""Multi-level mask generation (K3), the compact plan, and budget accounting.

Drop-ins for pkg/src/pyrattn/mask.py :
  assign_threshold :128-151, binary_mask :154-158, assign_quantile :167-179,
  combine_mask :237-247, causal_premask :324-349,
  SparsityReport / report_from_counts / sparsity_report :250-321.
Level assignment and plan emission run in libpsa (psa_assign_levels); the report is exact
rational arithmetic on the host from device-side level counts, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import torch

from . import _lib
from ._tensors import require_cuda, stream_handle, to_device
from .errors import ValidationError
from .layout import BlockLayout, LevelThresholds, QuantileCutpoints


@dataclass
class MaskPlan:
    """Level map plus the per-(head, query block) selected-block lists the attention kernel
    walks (level-major, ascending block index within a level)."""

    level_map: torch.Tensor      # int8 [B, Hq, n_q, n_k]
    csr: torch.Tensor            # uint16-as-int16 [B*Hq*n_q, n_k]: j | level << 12
    info: torch.Tensor           # int32 [B*Hq*n_q, 2]: (entries, total power-of-two slot rows)
    level_counts: torch.Tensor   # int64 [levels+1] (device)
    levels: int

    def report(self) -> "SparsityReport":
        counts = [int(c) for c in self.level_counts.cpu().tolist()]
        return report_from_counts(counts, sum(counts))

    def selected_blocks(self, unit: int) -> list:
        """Selected (j, level) pairs of one work unit, level-major (for inspection/tests)."""
        n = int(self.info[unit, 0])
        ent = self.csr[unit, :n].to(torch.int32).cpu().tolist()
        return [((e & 0xFFFF) & 0xFFF, (e & 0xFFFF) >> 12) for e in ent]


def _alloc_plan(B: int, Hq: int, n_q: int, n_k: int, levels: int, dev) -> MaskPlan:
    units = B * Hq * n_q
    return MaskPlan(
        level_map=torch.empty(B, Hq, n_q, n_k, dtype=torch.int8, device=dev),
        csr=torch.empty(units, n_k, dtype=torch.int16, device=dev),
        info=torch.empty(units, 2, dtype=torch.int32, device=dev),
        level_counts=torch.zeros(levels + 1, dtype=torch.int64, device=dev),
        levels=levels,
    )


def assign_levels_device(scores: torch.Tensor, *, mode: str, rule, levels: int,
                         b_q: int = 1, b_k: int = 1, hkv: int | None = None,
                         caps: torch.Tensor | None = None, causal: bool = False,
                         qblocks: torch.Tensor | None = None) -> MaskPlan:
    """scores fp64 [B, Hq, n_q, n_k] (device) -> MaskPlan. ``rule`` is LevelThresholds
    (mode 'threshold') or QuantileCutpoints (mode 'quantile'). ``qblocks`` (device int32
    [n_q]): score row i is query block qblocks[i] of the head (q-block work units)."""
    B, Hq, n_q, n_k = scores.shape
    hkv = Hq if hkv is None else hkv
    dev = scores.device
    if len(rule) > levels:
        raise ValidationError(f"{len(rule)} thresholds exceed {levels} levels")
    plan = _alloc_plan(B, Hq, n_q, n_k, levels, dev)
    if mode == "threshold":
        taus, counts, m = _lib.host_doubles(rule.taus), None, 0
    else:
        taus, counts, m = None, _lib.host_ints(rule.counts(n_k)), 1
    if qblocks is not None and qblocks.numel() != n_q:
        raise ValidationError(f"{qblocks.numel()} query blocks for {n_q} score rows")
    rc = _lib.load().psa_assign_levels_rows(
        scores.data_ptr(), B, Hq, hkv, n_q, n_k, m, taus, counts, len(rule),
        _lib.ptr(caps), int(causal), b_q, b_k, levels, _lib.ptr(qblocks),
        plan.level_map.data_ptr(), plan.csr.data_ptr(), plan.info.data_ptr(),
        plan.level_counts.data_ptr(), stream_handle(dev))
    _lib.check(rc, "psa_assign_levels")
    return plan


def plan_from_mask(mask: torch.Tensor, layout: BlockLayout, causal: bool,
                   batch: int, hq: int) -> MaskPlan:
    """Plan for a caller-supplied level map (validated like attention.py:66-108)."""
    require_cuda(mask, "mask")
    m = mask
    if m.dtype not in (torch.int8, torch.int64):
        m = m.to(torch.int64)
    m = m.reshape(batch, hq, layout.n_q, layout.n_k).contiguous()
    dev = m.device
    plan = _alloc_plan(batch, hq, layout.n_q, layout.n_k, layout.levels, dev)
    plan.level_map = m if m.dtype == torch.int8 else m.to(torch.int8)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = _lib.load().psa_mask_to_plan(
        m.data_ptr(), int(m.dtype == torch.int64), batch * hq * layout.n_q, layout.n_q,
        layout.n_k, int(causal), layout.q_block, layout.k_block, layout.levels,
        plan.csr.data_ptr(), plan.info.data_ptr(), plan.level_counts.data_ptr(),
        bad.data_ptr(), stream_handle(dev))
    _lib.check(rc, "psa_mask_to_plan")
    flag = int(bad.item())
    if flag & 1:
        raise ValidationError(f"mask levels outside 0..{layout.levels}")
    if flag & 2:
        raise ValidationError("causal mode requires level 1 on straddling pairs; run the mask "
                              "through the causal pre-pass first")
    return plan


def _check_scores(scores) -> tuple:
    scores = to_device(scores, "importance scores")
    if scores.ndim < 2 or scores.numel() == 0:
        raise ValidationError("importance scores must be a non-empty matrix")
    s = scores.to(torch.float64)
    if not bool(torch.isfinite(s).all()):
        raise ValidationError("importance scores contains NaN or Inf entries")
    if bool((s < 0).any()):
        raise ValidationError("importance scores must be non-negative")
    lead = tuple(s.shape[:-2])
    s4 = s.reshape((1,) * (4 - s.ndim) + tuple(s.shape)) if s.ndim <= 4 else None
    if s4 is None:
        raise ValidationError("scores must have at most 4 dims")
    return s4.contiguous(), lead


def assign_threshold(scores, thresholds: LevelThresholds) -> torch.Tensor:
    """Alg. 2 level assignment (mask.py:128-151); int64, same shape as ``scores``."""
    s4, lead = _check_scores(scores)
    plan = assign_levels_device(s4, mode="threshold", rule=thresholds, levels=len(thresholds))
    return plan.level_map.to(torch.int64).reshape(lead + tuple(s4.shape[2:]))


def binary_mask(scores, tau: float) -> torch.Tensor:
    """0/1 keep/drop mask (mask.py:154-158)."""
    if not 0.0 <= tau <= 1.0:
        raise ValidationError(f"tau must lie in [0, 1], got {tau}")
    return assign_threshold(scores, LevelThresholds((tau,)))


def assign_quantile(scores, cutpoints: QuantileCutpoints) -> torch.Tensor:
    """Rank-fraction level assignment (mask.py:167-179); int64."""
    s4, lead = _check_scores(scores)
    plan = assign_levels_device(s4, mode="quantile", rule=cutpoints, levels=len(cutpoints))
    return plan.level_map.to(torch.int64).reshape(lead + tuple(s4.shape[2:]))


def combine_mask(mask, caps) -> torch.Tensor:
    """min(M, caps[j]) with zeros kept (mask.py:237-247). Elementwise on the device."""
    mask = to_device(mask, "mask")
    caps = to_device(caps, "caps")
    m = mask.to(torch.int64)
    c = caps.to(torch.int64)
    if m.ndim < 2 or c.ndim < 1 or m.shape[-1] != c.shape[-1]:
        raise ValidationError(f"mask columns {tuple(m.shape)} must match cap length {tuple(c.shape)}")
    if bool((c < 1).any()):
        raise ValidationError("level caps must be >= 1")
    return torch.minimum(m, c.unsqueeze(-2))


def causal_premask(mask, layout: BlockLayout) -> torch.Tensor:
    """Causal pre-pass (mask.py:324-349): future -> 0, straddling -> 1, visible -> keep."""
    mask = to_device(mask, "mask")
    m = mask.to(torch.int64)
    if tuple(m.shape[-2:]) != (layout.n_q, layout.n_k):
        raise ValidationError(f"mask shape {tuple(m.shape)} does not match layout "
                              f"{(layout.n_q, layout.n_k)}")
    dev = m.device
    i = torch.arange(layout.n_q, device=dev)[:, None]
    j = torch.arange(layout.n_k, device=dev)[None, :]
    future = j * layout.k_block > (i + 1) * layout.q_block - 1
    visible = (j + 1) * layout.k_block - 1 <= i * layout.q_block
    out = torch.where(future, torch.zeros_like(m), m)
    return torch.where(~future & ~visible, torch.ones_like(m), out)


@dataclass(frozen=True)
class SparsityReport:
    """Compute-budget accounting of one mask; floats are exact rationals rounded once."""

    level_counts: tuple
    total: int
    rho_bar: float
    sparsity: float
    kv_coverage: float
    level_histogram: tuple

    def as_dict(self) -> dict:
        return {
            "level_counts": list(self.level_counts),
            "total_entries": self.total,
            "rho_bar": self.rho_bar,
            "sparsity": self.sparsity,
            "kv_coverage": self.kv_coverage,
            "level_histogram": list(self.level_histogram),
        }


def report_from_counts(level_counts, total: int) -> SparsityReport:
    """SparsityReport from per-level counts: rho = sum_h counts_h/total * 2^(1-h), exact."""
    counts = tuple(int(c) for c in level_counts)
    if total < 1 or any(c < 0 for c in counts) or sum(counts) != total:
        raise ValidationError("level counts must be non-negative and sum to total")
    rho = sum((Fraction(counts[h], total) / (1 << (h - 1)) for h in range(1, len(counts))),
              Fraction(0))
    return SparsityReport(
        level_counts=counts, total=total, rho_bar=float(rho), sparsity=float(1 - rho),
        kv_coverage=float(Fraction(total - counts[0], total)),
        level_histogram=tuple(float(Fraction(c, total)) for c in counts))


def sparsity_report(mask, levels: int | None = None) -> SparsityReport:
    """Budget, sparsity and coverage of a level map (mask.py:303-321)."""
    m = (to_device(mask, "mask") if torch.cuda.is_available() else torch.as_tensor(mask)).to(torch.int64)
    if m.ndim < 2 or m.numel() == 0:
        raise ValidationError("mask must be a non-empty 2D integer array")
    if bool((m < 0).any()):
        raise ValidationError("mask levels must be >= 0")
    top = int(m.max())
    lv = max(top if levels is None else int(levels), 1)
    if top > lv:
        raise ValidationError(f"mask contains level {top} > levels={lv}")
    counts = torch.bincount(m.reshape(-1), minlength=lv + 1).cpu().tolist()
    return report_from_counts(counts, m.numel())

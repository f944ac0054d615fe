"""The fused PSA forward: the reference's per-head stage order (pipeline._run_head,
pkg/src/pyrattn/pipeline.py:256-314) run for every (batch, head) at once on the GPU:

  pyramid (K1) -> importance (K2, non-causal) -> level assignment (K3) [-> similarity cap]
  [-> causal pre-pass] -> multi-level attention (K4)

The reference's optional space-filling-curve permutation (``grid``/``unpermute``) runs as
row gathers in libpsa; the dense oracle of the reference run is not part of this operator
(see DESIGN.md). ``RunConfig`` keeps the reference's flat key
names and validation (pipeline.py:38-137) so existing JSON configs drive the GPU path.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, fields

import torch

from ._tensors import as_bhnd, restore
from .attention import attention_forward
from .errors import NumericError, ValidationError
from .importance import antidiagonal_scores, importance_scores
from .layout import (PRESET_CUTPOINTS, LevelThresholds, QuantileCutpoints, SamplerConfig,
                     SimThresholds, make_layout)
from .mask import MaskPlan, assign_levels_device
from .permute import gather_rows, hilbert_order
from .pyramid import PyramidKV, build_pyramid, similarity_caps

ESTIMATORS = ("sampled-max", "sampled-mean", "antidiagonal")
MASK_STRATEGIES = ("threshold", "quantile", "binary") + tuple(PRESET_CUTPOINTS)


@dataclass(frozen=True)
class RunConfig:
    """Flat run description with the reference's keys (pipeline.py:38-62)."""

    n: int
    d: int
    b_q: int
    b_k: int
    levels: int
    estimator: str
    mask: str
    tile_len: int
    grid: tuple | None = None
    s_q: int | None = None
    s_k: int | None = None
    stride: int | None = None
    seed: int | None = None
    thresholds: tuple | None = None
    cutpoints: tuple | None = None
    tau: float | None = None
    sim_thresholds: tuple | None = None
    causal: bool = False
    num_steps: int = 1
    dense_prefix: float = 0.0
    unpermute: bool = False

    def __post_init__(self):
        if self.estimator not in ESTIMATORS:
            raise ValidationError(f"estimator {self.estimator!r} not one of {ESTIMATORS}")
        if self.mask not in MASK_STRATEGIES:
            raise ValidationError(f"mask strategy {self.mask!r} not one of {MASK_STRATEGIES}")
        if self.estimator.startswith("sampled"):
            if self.s_q is None or self.s_k is None:
                raise ValidationError("sampled estimators need s_q and s_k")
            if self.seed is None:
                raise ValidationError("sampled estimators need an explicit seed")
        if self.estimator == "antidiagonal" and self.stride is None:
            raise ValidationError("antidiagonal estimator needs a stride")
        need = {"threshold": "thresholds", "quantile": "cutpoints", "binary": "tau"}
        if self.mask in need:
            val = getattr(self, need[self.mask])
            if val is None or (self.mask != "binary" and not val):
                raise ValidationError(f"{self.mask} strategy needs {need[self.mask]}")
        if self.tile_len < 1:
            raise ValidationError("tile_len must be >= 1")
        if self.num_steps < 1:
            raise ValidationError("num_steps must be >= 1")
        if not 0.0 <= self.dense_prefix <= 1.0:
            raise ValidationError("dense_prefix must lie in [0, 1]")
        if self.grid is not None:
            grid = tuple(int(g) for g in self.grid)
            if math.prod(grid) != self.n:
                raise ValidationError(f"grid {grid} covers {math.prod(grid)} tokens, expected {self.n}")
            object.__setattr__(self, "grid", grid)
        for name in ("thresholds", "cutpoints", "sim_thresholds"):
            val = getattr(self, name)
            if val is not None:
                object.__setattr__(self, name, tuple(float(x) for x in val))

    @classmethod
    def from_dict(cls, data: dict) -> "RunConfig":
        known = {f.name for f in fields(cls)}
        unknown = set(data) - known
        if unknown:
            raise ValidationError(f"unknown config keys: {sorted(unknown)}")
        missing = {"n", "d", "b_q", "b_k", "levels", "estimator", "mask", "tile_len"} - set(data)
        if missing:
            raise ValidationError(f"missing config keys: {sorted(missing)}")
        data = dict(data)
        if data.get("sim_thresholds") == "off":
            data["sim_thresholds"] = None
        return cls(**data)

    @classmethod
    def from_json(cls, path) -> "RunConfig":
        with open(path, "r", encoding="utf-8") as fh:
            data = json.load(fh)
        if not isinstance(data, dict):
            raise ValidationError("config file must hold a JSON object")
        return cls.from_dict(data)

    def to_dict(self) -> dict:
        return {f.name: (list(v) if isinstance(v := getattr(self, f.name), tuple) else v)
                for f in fields(self)}

    def layout(self):
        return make_layout(self.n, self.d, self.b_q, self.b_k, self.levels)


@dataclass
class PSAResult:
    out: torch.Tensor            # bf16, q's shape
    lse: torch.Tensor            # fp32 natural-log normalisers
    plan: MaskPlan               # level map + selected-block lists + level counts
    skipped: torch.Tensor        # device int32 counter of rows with no key
    scores: torch.Tensor | None  # fp64 importance (kept when requested)
    pyramid: PyramidKV | None

    @property
    def level_map(self) -> torch.Tensor:
        return self.plan.level_map

    def sparsity(self):
        return self.plan.report()

    def skipped_rows(self) -> int:
        return int(self.skipped.item())


def _stage(name: str, fn, *args, **kw):
    try:
        return fn(*args, **kw)
    except (ValidationError, NumericError) as exc:  # same tagging as pipeline.py:247-253
        raise type(exc)(f"[stage: {name}] {exc}") from exc


def _mask_rule(cfg: RunConfig, levels: int):
    if cfg.mask == "threshold":
        rule = LevelThresholds(cfg.thresholds)
        if len(rule) > levels:
            raise ValidationError(f"{len(rule)} thresholds exceed {levels} levels")
        return "threshold", rule
    if cfg.mask == "binary":
        if not 0.0 <= cfg.tau <= 1.0:
            raise ValidationError(f"tau must lie in [0, 1], got {cfg.tau}")
        return "threshold", LevelThresholds((cfg.tau,))
    rule = QuantileCutpoints(cfg.cutpoints) if cfg.mask == "quantile" else PRESET_CUTPOINTS[cfg.mask]
    if len(rule) > levels:
        raise ValidationError(f"{len(rule)} cutpoints exceed {levels} levels "
                              "(presets need levels >= 4)")
    return "quantile", rule


def psa_forward_4d(q4, k4, v4, cfg: RunConfig, keep_scores: bool = False,
                   out: torch.Tensor | None = None, lse: torch.Tensor | None = None) -> PSAResult:
    """Fused PSA forward on contiguous bf16 [B, H, N, d] device tensors (``out``/``lse``:
    optional preallocated device outputs)."""
    lay = cfg.layout()
    lay.check_gpu()
    perm = None
    if cfg.grid is not None:  # pipeline.py:257-263: curve order applied to Q, K and V
        perm = _stage("permutation", hilbert_order, cfg.grid)
        order, _ = perm.on(q4.device)
        q4, k4, v4 = (gather_rows(x, order) for x in (q4, k4, v4))
        final_out, final_lse = out, lse
        out = lse = None
    mode, rule = _mask_rule(cfg, lay.levels)
    B, Hq = q4.shape[:2]
    Hkv = k4.shape[1]
    pyr = _stage("pyramid", build_pyramid, k4, v4, lay)
    if cfg.estimator == "antidiagonal":  # pipeline._estimate (pipeline.py:239-244)
        scores = _stage("importance", antidiagonal_scores, q4, k4, lay, cfg.stride)
    else:
        sampler = SamplerConfig(s_q=cfg.s_q, s_k=cfg.s_k, seed=cfg.seed)
        reducer = "max" if cfg.estimator == "sampled-max" else "mean"
        scores = _stage("importance", importance_scores, q4, k4, lay, sampler, reducer)
    caps = None
    if cfg.sim_thresholds is not None:
        caps = _stage("similarity-cap", similarity_caps, k4, lay, SimThresholds(cfg.sim_thresholds))
    plan = _stage("mask", assign_levels_device, scores, mode=mode, rule=rule, levels=lay.levels,
                  b_q=lay.q_block, b_k=lay.k_block, hkv=Hkv, caps=caps, causal=cfg.causal)
    out, lse, skipped = _stage("executor", attention_forward, q4, pyr, plan, cfg.causal, out, lse)
    if perm is not None:
        if cfg.unpermute:  # pipeline.py:312-313: back to the caller's token order
            _, inverse = perm.on(q4.device)
            out = gather_rows(out, inverse, final_out)
            lse = gather_rows(lse.unsqueeze(-1), inverse,
                              None if final_lse is None else final_lse.unsqueeze(-1)).squeeze(-1)
        else:
            if final_out is not None:
                final_out.copy_(out)
                out = final_out
            if final_lse is not None:
                final_lse.copy_(lse)
                lse = final_lse
    return PSAResult(out=out, lse=lse, plan=plan, skipped=skipped,
                     scores=scores if keep_scores else None, pyramid=pyr)


def resolve_config(cfg: RunConfig | None, n: int, d: int, overrides: dict) -> RunConfig:
    """RunConfig from an explicit config and/or keyword overrides; n, d from the tensors."""
    if cfg is None:
        data = {"n": n, "d": d, "tile_len": 128}
        data.update(overrides)
        cfg = RunConfig.from_dict(data)
    elif overrides:
        cfg = RunConfig.from_dict({**cfg.to_dict(), **overrides})
    if (cfg.n, cfg.d) != (n, d):
        raise ValidationError(f"tensor shape {(n, d)} does not match config ({cfg.n}, {cfg.d})")
    return cfg


def psa_attention(q, k, v, cfg: RunConfig | None = None, *, keep_scores: bool = False,
                  **overrides) -> PSAResult:
    """Pyramid sparse attention forward.

    ``q``: (n, d), (Hq, n, d) or (B, Hq, n, d); ``k``/``v``: same with Hkv heads (Hq % Hkv == 0).
    Configuration by ``RunConfig`` or its keys as keyword arguments (n and d are taken from
    the tensors; tile_len defaults to 128).

    CUDA tensors run in place on their device. Host tensors (ideally pinned) go through
    ``staging.psa_attention_staged``: head groups are copied in, computed and copied back on
    three overlapped streams, and the result lives in host memory (the reference's
    arrays-in/arrays-out contract); the compute is the same sm_100a path, never a CPU one.
    """
    if isinstance(q, torch.Tensor) and not q.is_cuda:
        from .staging import psa_attention_staged  # host tensors: pipelined staging onto the GPU
        return psa_attention_staged(q, k, v, cfg, keep_scores=keep_scores, **overrides)
    q4, lead = as_bhnd(q, "Q")
    k4, _ = as_bhnd(k, "K", q4.shape[2], q4.shape[3])
    v4, _ = as_bhnd(v, "V", q4.shape[2], q4.shape[3])
    if k4.shape != v4.shape or k4.shape[0] != q4.shape[0]:
        raise ValidationError(f"Q/K/V shapes differ: {tuple(q4.shape)}/{tuple(k4.shape)}/"
                              f"{tuple(v4.shape)}")
    cfg = resolve_config(cfg, q4.shape[2], q4.shape[3], overrides)
    res = psa_forward_4d(q4, k4, v4, cfg, keep_scores=keep_scores)
    res.out = restore(res.out, lead)
    res.lse = res.lse.reshape(lead + (cfg.n,))
    return res

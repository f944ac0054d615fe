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
import os
from dataclasses import dataclass, fields

import torch

from ._tensors import as_bhnd, restore
from .attention import attention_forward
from .errors import NumericError, ValidationError
from .importance import antidiagonal_scores, importance_scores, query_blocks
from .layout import (PRESET_CUTPOINTS, LevelThresholds, QuantileCutpoints, SamplerConfig,
                     SimThresholds, make_layout)
from .mask import MaskPlan, assign_levels_device
from .permute import gather_rows, hilbert_order
from .pyramid import PyramidKV, build_pyramid, build_pyramid_gather, similarity_caps

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
    nonfinite: torch.Tensor | None = None  # device int32 [1]: Q/K/V held NaN/Inf (check_finite)

    @property
    def level_map(self) -> torch.Tensor:
        return self.plan.level_map

    def sparsity(self):
        return self.plan.report()

    def skipped_rows(self) -> int:
        return int(self.skipped.item())


_NVTX = os.environ.get("PSA_NVTX", "0") not in ("", "0")


def _stage(name: str, fn, *args, **kw):
    """One stage of the fused call: errors tagged like pipeline.py:247-253; with PSA_NVTX=1 the
    stage is an NVTX range (``psa:<stage>``) for nsys / ncu --nvtx timelines."""
    if _NVTX:
        torch.cuda.nvtx.range_push(f"psa:{name}")
    try:
        return fn(*args, **kw)
    except (ValidationError, NumericError) as exc:  # same tagging as pipeline.py:247-253
        raise type(exc)(f"[stage: {name}] {exc}") from exc
    finally:
        if _NVTX:
            torch.cuda.nvtx.range_pop()


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
                   out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                   qblocks=None, check_finite: bool = False) -> PSAResult:
    """Fused PSA forward on contiguous bf16 [B, H, N, d] device tensors (``out``/``lse``:
    optional preallocated device outputs). ``qblocks``: run only these query blocks of every
    head (a (b, h, q-block set) work unit of parallel.py); importance rows, level map, plan, O
    and lse then hold those blocks in that order (compact), each identical to the full call's."""
    lay = cfg.layout()
    lay.check_gpu()
    blk = _stage("partition", query_blocks, qblocks, lay, q4.device)
    if blk is not None and cfg.grid is not None:
        raise ValidationError("query-block subsets are not supported with grid permutations")
    perm = order = None
    bad = None
    if check_finite:  # linalg.py:15-24 (as_matrix): device flag, raised by the caller after a sync
        bad = (~torch.isfinite(q4)).any().to(torch.int32).reshape(1)
    if cfg.grid is not None:  # pipeline.py:257-263: curve order applied to Q, K and V
        perm = _stage("permutation", hilbert_order, cfg.grid)
        order, _ = perm.on(q4.device)
        q4 = gather_rows(q4, order)
        # K/V: the gather is fused into the pyramid kernel's loads (level 1 = permuted K/V)
        if bad is not None:
            bad |= ((~torch.isfinite(k4)).any() | (~torch.isfinite(v4)).any()).to(torch.int32)
        pyr = _stage("pyramid", build_pyramid_gather, k4, v4, lay, order)
        k4, v4 = pyr.k_raw, pyr.v_raw
    else:
        pyr = _stage("pyramid", build_pyramid, k4, v4, lay, flag=bad)
    mode, rule = _mask_rule(cfg, lay.levels)
    B, Hq = q4.shape[:2]
    Hkv = k4.shape[1]
    if cfg.estimator == "antidiagonal":  # pipeline._estimate (pipeline.py:239-244)
        scores = _stage("importance", antidiagonal_scores, q4, k4, lay, cfg.stride, qblocks=blk)
    else:
        sampler = SamplerConfig(s_q=cfg.s_q, s_k=cfg.s_k, seed=cfg.seed)
        reducer = "max" if cfg.estimator == "sampled-max" else "mean"
        scores = _stage("importance", importance_scores, q4, k4, lay, sampler, reducer,
                        qblocks=blk)
    caps = None
    if cfg.sim_thresholds is not None:
        caps = _stage("similarity-cap", similarity_caps, k4, lay, SimThresholds(cfg.sim_thresholds))
    plan = _stage("mask", assign_levels_device, scores, mode=mode, rule=rule, levels=lay.levels,
                  b_q=lay.q_block, b_k=lay.k_block, hkv=Hkv, caps=caps, causal=cfg.causal,
                  qblocks=blk)
    # pipeline.py:312-313 (back to the caller's token order) fused into the attention epilogue
    scatter = order if perm is not None and cfg.unpermute else None
    out, lse, skipped = _stage("executor", attention_forward, q4, pyr, plan, cfg.causal, out, lse,
                               None, scatter, blk)
    return PSAResult(out=out, lse=lse, plan=plan, skipped=skipped,
                     scores=scores if keep_scores else None, pyramid=pyr, nonfinite=bad)


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
                  qblocks=None, check_finite: bool = True, **overrides) -> PSAResult:
    """Pyramid sparse attention forward.

    ``q``: (n, d), (Hq, n, d) or (B, Hq, n, d); ``k``/``v``: same with Hkv heads (Hq % Hkv == 0).
    Configuration by ``RunConfig`` or its keys as keyword arguments (n and d are taken from
    the tensors; tile_len defaults to 128).

    CUDA tensors run in place on their device. Host tensors (ideally pinned) go through
    ``staging.psa_attention_staged``: head groups are copied in, computed and copied back on
    three overlapped streams, and the result lives in host memory (the reference's
    arrays-in/arrays-out contract); the compute is the same sm_100a path, never a CPU one.
    ``qblocks``: only these query blocks of every head (a work unit of parallel.partition); the
    outputs then hold those blocks' rows (compact). ``check_finite``: NaN/Inf in Q, K or V
    raise ValidationError like the reference's as_matrix (linalg.py:15-24); the K/V test rides in
    the pyramid kernel's loads, the Q test is one reduction, both read after the forward (one
    host sync per call).
    """
    if not isinstance(q, torch.Tensor):  # array-likes (as_matrix, linalg.py:15-24): host tensors
        import numpy as np
        q, k, v = (torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
                   for x in (q, k, v))
    if isinstance(q, torch.Tensor) and not q.is_cuda:
        from .staging import psa_attention_staged  # host tensors: pipelined staging onto the GPU
        return psa_attention_staged(q, k, v, cfg, keep_scores=keep_scores, qblocks=qblocks,
                                    check_finite=check_finite, **overrides)
    q4, lead = as_bhnd(q, "Q")
    k4, _ = as_bhnd(k, "K", q4.shape[2], q4.shape[3])
    v4, _ = as_bhnd(v, "V", q4.shape[2], q4.shape[3])
    if k4.shape != v4.shape or k4.shape[0] != q4.shape[0]:
        raise ValidationError(f"Q/K/V shapes differ: {tuple(q4.shape)}/{tuple(k4.shape)}/"
                              f"{tuple(v4.shape)}")
    cfg = resolve_config(cfg, q4.shape[2], q4.shape[3], overrides)
    res = psa_forward_4d(q4, k4, v4, cfg, keep_scores=keep_scores, qblocks=qblocks,
                         check_finite=check_finite)
    if res.nonfinite is not None and int(res.nonfinite.item()):
        raise ValidationError("[stage: input] Q, K or V contains NaN or Inf entries")
    rows = res.out.shape[2]
    res.out = res.out.reshape(lead + (rows, q4.shape[3]))
    res.lse = res.lse.reshape(lead + (rows,))
    return res


# ------------------------------------------------------------------ run_pipeline (report API)
@dataclass
class PipelineResult:
    report: dict
    output: object  # attention output, same container (torch / numpy) and leading dims as q


def relative_error(a: torch.Tensor, b: torch.Tensor) -> float:
    """Frobenius ||a - b|| / ||b|| (linalg.py:61-70), computed on the device in fp32."""
    den = torch.linalg.vector_norm(b.float())
    if float(den) == 0.0:
        raise NumericError("relative error undefined for a zero-norm reference")
    return float(torch.linalg.vector_norm(a.float() - b.float()) / den)


def _steps_metadata(cfg: RunConfig, rho_bar: float) -> dict:
    """pipeline.py:317-330."""
    dense = min(math.ceil(cfg.dense_prefix * cfg.num_steps) if cfg.dense_prefix > 0 else 0,
                cfg.num_steps)
    modes = ["dense"] * dense + ["sparse"] * (cfg.num_steps - dense)
    return {"num_steps": cfg.num_steps, "dense_prefix": cfg.dense_prefix, "dense_steps": dense,
            "modes": modes,
            "mean_rho_over_steps": (dense * 1.0 + (cfg.num_steps - dense) * rho_bar) / cfg.num_steps}


def run_pipeline(cfg: RunConfig, q, k, v) -> PipelineResult:
    """pipeline.py:333-397 on the GPU: every head at once through psa_forward_4d, then the
    reference's report (per-head sparsity, schedule utilisation for tile_len, error against
    dense attention, skipped rows, steps metadata, aggregates). Inputs: (n, d) or (heads, n, d)
    torch tensors or numpy arrays (moved to the current CUDA device as bf16); the output has
    the input's container type. The dense baseline is the same sm_100a kernel with every block
    at level 1 (bf16), and the tiled ("schedule") execution is the kernel itself, so
    schedule_relative_error equals relative_error."""
    import time

    import numpy as np

    from .attention import causal_full_attention, full_attention
    from .mask import report_from_counts

    t0 = time.perf_counter()
    is_np = not isinstance(q, torch.Tensor)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if dev is None:
        raise ValidationError("run_pipeline needs a CUDA device (no CPU fallback)")

    def to_dev(x):
        x = torch.from_numpy(np.ascontiguousarray(x)) if not isinstance(x, torch.Tensor) else x
        return x.to(dev, torch.bfloat16)

    q, k, v = to_dev(q), to_dev(k), to_dev(v)
    if q.shape != k.shape or k.shape != v.shape:
        raise ValidationError(f"Q/K/V shapes differ: {tuple(q.shape)}/{tuple(k.shape)}/"
                              f"{tuple(v.shape)}")
    if q.ndim not in (2, 3):
        raise ValidationError(f"expected (n, d) or (heads, n, d), got {tuple(q.shape)}")
    squeeze = q.ndim == 2
    q3, k3, v3 = (x.unsqueeze(0) if squeeze else x for x in (q, k, v))
    if tuple(q3.shape[1:]) != (cfg.n, cfg.d):
        raise ValidationError(f"tensor shape {tuple(q3.shape[1:])} does not match config "
                              f"({cfg.n}, {cfg.d})")
    lay = cfg.layout()
    heads = q3.shape[0]
    res = psa_forward_4d(q3[None].contiguous(), k3[None].contiguous(), v3[None].contiguous(), cfg)
    out = res.out[0]
    lm = res.plan.level_map[0].to(torch.int64)  # [heads, n_q, n_k]
    dense_fn = causal_full_attention if cfg.causal else full_attention
    if cfg.grid is not None:  # the dense oracle sees the same (permuted) token order
        from .permute import apply_permutation, hilbert_order
        p = hilbert_order(cfg.grid)
        qd, kd, vd = (apply_permutation(x, p) for x in (q3, k3, v3))
    else:
        qd, kd, vd = q3, k3, v3
    dense = dense_fn(qd, kd, vd).out
    if cfg.grid is not None and cfg.unpermute:
        from .permute import apply_permutation, hilbert_order, invert_permutation
        dense = apply_permutation(dense, invert_permutation(hilbert_order(cfg.grid)))
    pooled = torch.tensor([0] + [lay.pooled_len(h) for h in range(1, lay.levels + 1)],
                          dtype=torch.int64, device=lm.device)
    rows_qb = pooled[lm].sum(dim=2)                               # [heads, n_q]
    tiles_qb = (rows_qb + cfg.tile_len - 1) // cfg.tile_len       # greedy merge packing
    counts = torch.stack([(lm == h).sum(dim=(1, 2)) for h in range(lay.levels + 1)], dim=1)
    skipped_h = (~torch.isfinite(res.lse[0])).sum(dim=1)
    counts, rows_h, tiles_h, skipped_h = (x.cpu().tolist() for x in
                                          (counts, rows_qb.sum(1), tiles_qb.sum(1), skipped_h))
    per_head = []
    for h in range(heads):
        err = relative_error(out[h], dense[h])
        cap = tiles_h[h] * cfg.tile_len
        per_head.append({
            "relative_error": err, "schedule_relative_error": err,
            "sparsity": report_from_counts(counts[h], lay.n_q * lay.n_k).as_dict(),
            "utilization": {"tiles": tiles_h[h], "useful_rows": rows_h[h], "capacity": cap,
                            "utilization": rows_h[h] / cap if cap else 1.0},
            "selected_pooled_rows": rows_h[h], "skipped_rows": skipped_h[h]})
    tot_counts = [sum(c[i] for c in counts) for i in range(lay.levels + 1)]
    agg = report_from_counts(tot_counts, heads * lay.n_q * lay.n_k).as_dict()
    tiles, useful = sum(tiles_h), sum(rows_h)
    capacity = tiles * cfg.tile_len
    report = {
        "config": cfg.to_dict(), "heads": heads,
        "relative_error": float(np.mean([h["relative_error"] for h in per_head])),
        "schedule_relative_error": float(np.mean([h["schedule_relative_error"] for h in per_head])),
        "sparsity": agg,
        "utilization": {"tiles": tiles, "useful_rows": useful, "capacity": capacity,
                        "utilization": useful / capacity if capacity else 1.0},
        "skipped_rows": sum(skipped_h), "per_head": per_head,
        "steps": _steps_metadata(cfg, agg["rho_bar"]),
        "wall_time_s": time.perf_counter() - t0,
    }
    output = out[0] if squeeze else out
    if is_np:
        output = output.float().cpu().numpy()
    return PipelineResult(report=report, output=output)


def report_to_json(report: dict) -> str:
    """Deterministic JSON rendering (pipeline.py:400-402)."""
    return json.dumps(report, sort_keys=True, indent=2) + "\n"

"""Host-resident PSA forward: arrays in, arrays out, like the reference's run_pipeline
(pkg/src/pyrattn/pipeline.py:333-397 takes and returns host arrays), with every tensor
operation on the GPU.

Q/K/V stay in (pinned) host memory; the call walks groups of KV heads (with their GQA query
heads) through three CUDA streams so PCIe traffic overlaps the kernels:

    copy-in stream   H2D of group g+1 ─┐
    compute stream   PSA forward of group g (pyramid → importance → levels → attention)
    copy-out stream  D2H of O / lse of group g-1

Two device slots per tensor double-buffer the groups; events order slot reuse. Every group runs
the same kernels on the same per-head inputs as the device-resident path, so results are
bit-identical to ``psa_attention`` on CUDA tensors (tests/test_gpu_parity.py). Nothing here
computes on the CPU: without a CUDA device the call raises.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .errors import ValidationError
from .mask import SparsityReport, report_from_counts


@dataclass
class StagedResult:
    """Result of a host-resident forward: ``out`` bf16 and ``lse`` fp32 in host memory."""

    out: torch.Tensor
    lse: torch.Tensor
    level_counts: list = field(default_factory=list)
    skipped: int = 0
    level_map: torch.Tensor | None = None   # int8 [B, Hq, n_q, n_k] on the host when requested

    def sparsity(self) -> SparsityReport:
        return report_from_counts(self.level_counts, sum(self.level_counts))

    def skipped_rows(self) -> int:
        return self.skipped


def _host_bhnd(x, name: str):
    if not isinstance(x, torch.Tensor):
        raise ValidationError(f"{name} must be a torch.Tensor")
    if x.is_cuda:
        raise ValidationError(f"{name}: staged path expects host tensors")
    if x.ndim not in (2, 3, 4) or x.numel() == 0:
        raise ValidationError(f"{name} must be a non-empty (n, d), (heads, n, d) or "
                              f"(batch, heads, n, d) tensor, got shape {tuple(x.shape)}")
    if not x.is_floating_point():
        raise ValidationError(f"{name} must be a floating-point tensor")
    lead = tuple(x.shape[:-2])
    x4 = x.reshape((1,) * (4 - x.ndim) + tuple(x.shape))
    if x4.dtype != torch.bfloat16:
        x4 = x4.to(torch.bfloat16)
    return x4.contiguous(), lead


def _group_sizes(n: int) -> list:
    """KV-head group sizes for one batch entry: about 20 equal groups. Small groups keep the
    copy-in, compute and copy-out streams overlapped down to the PCIe floor (cfg3, 40 KV heads:
    2 heads per group 46.9 ms, 3: 47.1, 1: 47.8, six groups of 6 then 3 and 1: 48.3, 8: 52.9;
    H2D alone 41.8 ms, H2D and D2H together 47.2 ms)."""
    per = max(1, -(-n // 20))
    return [min(per, n - i) for i in range(0, n, per)]


def psa_attention_staged(q, k, v, cfg=None, *, device=None, kv_heads_per_group: int | None = None,
                         out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                         keep_level_map: bool = False, keep_scores: bool = False,
                         qblocks=None, check_finite: bool = True, **overrides) -> StagedResult:
    """PSA forward of host tensors on ``device`` (default: the current CUDA device).

    ``out`` / ``lse``: optional preallocated (ideally pinned) host outputs of shapes
    q.shape and q.shape[:-1]. ``kv_heads_per_group``: pipeline granularity (default: about 20
    equal groups). Returns once the outputs are in host memory.
    """
    from .pipeline import psa_forward_4d, resolve_config

    if keep_scores:
        raise ValidationError("keep_scores is only available for device-resident inputs")
    if not torch.cuda.is_available():
        raise ValidationError("host tensors are staged onto a CUDA device and no CUDA device is "
                              "present: the sm_100a kernels are the only implementation (no CPU "
                              "fallback)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    q4, lead = _host_bhnd(q, "Q")
    k4, _ = _host_bhnd(k, "K")
    v4, _ = _host_bhnd(v, "V")
    B, Hq, n, d = q4.shape
    Hkv = k4.shape[1]
    if k4.shape != v4.shape or k4.shape[0] != B or k4.shape[2:] != q4.shape[2:] or Hq % Hkv:
        raise ValidationError(f"Q/K/V shapes differ: {tuple(q4.shape)}/{tuple(k4.shape)}/"
                              f"{tuple(v4.shape)}")
    cfg = resolve_config(cfg, n, d, overrides)
    lay = cfg.layout()
    group = Hq // Hkv
    # query-block work unit (parallel.partition): outputs hold the listed blocks' rows, compact
    n_sel = lay.n_q if qblocks is None else len(list(qblocks))
    rows = n_sel * lay.q_block
    if kv_heads_per_group is None:
        sizes = _group_sizes(Hkv) if B == 1 else [max(1, math.ceil(B * Hkv / 8))]
    else:
        sizes = [max(1, min(Hkv, int(kv_heads_per_group)))]
    g = max(sizes)

    if out is None:
        out = torch.empty(B, Hq, rows, d, dtype=torch.bfloat16, pin_memory=True)
    if lse is None:
        lse = torch.empty(B, Hq, rows, dtype=torch.float32, pin_memory=True)
    out4 = out.reshape(B, Hq, rows, d)
    lse3 = lse.reshape(B, Hq, rows)
    if out4.dtype != torch.bfloat16 or lse3.dtype != torch.float32 or out4.is_cuda or lse3.is_cuda:
        raise ValidationError("out must be a bf16 and lse an fp32 host tensor")
    lmap = (torch.empty(B, Hq, n_sel, lay.n_k, dtype=torch.int8, pin_memory=True)
            if keep_level_map else None)

    groups = []
    for b in range(B):
        h0, gi = 0, 0
        while h0 < Hkv:
            step = sizes[min(gi, len(sizes) - 1)]
            groups.append((b, h0, min(Hkv, h0 + step)))
            h0, gi = h0 + step, gi + 1
    with torch.cuda.device(dev):
        cur = torch.cuda.current_stream(dev)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        s_cmp = cur
        s_in.wait_stream(cur)
        slots = []
        for _ in range(min(2, len(groups))):
            slots.append({
                "q": torch.empty(1, g * group, n, d, dtype=torch.bfloat16, device=dev),
                "k": torch.empty(1, g, n, d, dtype=torch.bfloat16, device=dev),
                "v": torch.empty(1, g, n, d, dtype=torch.bfloat16, device=dev),
                "o": torch.empty(1, g * group, rows, d, dtype=torch.bfloat16, device=dev),
                "l": torch.empty(1, g * group, rows, dtype=torch.float32, device=dev),
                "free_in": None, "free_out": None,
            })
        counts = torch.zeros(lay.levels + 1, dtype=torch.int64, device=dev)
        skipped = torch.zeros(1, dtype=torch.int64, device=dev)
        bad = torch.zeros(1, dtype=torch.int64, device=dev)
        for gi, (b, h0, h1) in enumerate(groups):
            sl = slots[gi % len(slots)]
            nk, nq = h1 - h0, (h1 - h0) * group
            qs, ks, vs = sl["q"][:, :nq], sl["k"][:, :nk], sl["v"][:, :nk]
            os_, ls = sl["o"][:, :nq], sl["l"][:, :nq]
            with torch.cuda.stream(s_in):
                if sl["free_in"] is not None:
                    s_in.wait_event(sl["free_in"])
                qs.copy_(q4[b:b + 1, h0 * group:h1 * group], non_blocking=True)
                ks.copy_(k4[b:b + 1, h0:h1], non_blocking=True)
                vs.copy_(v4[b:b + 1, h0:h1], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(s_in)
            s_cmp.wait_event(ready)
            if sl["free_out"] is not None:
                s_cmp.wait_event(sl["free_out"])
            res = psa_forward_4d(qs, ks, vs, cfg, out=os_, lse=ls, qblocks=qblocks,
                                 check_finite=check_finite)
            counts += res.plan.level_counts
            skipped += res.skipped
            if res.nonfinite is not None:
                bad += res.nonfinite
            done = torch.cuda.Event()
            done.record(s_cmp)
            sl["free_in"] = done
            with torch.cuda.stream(s_out):
                s_out.wait_event(done)
                out4[b:b + 1, h0 * group:h1 * group].copy_(os_, non_blocking=True)
                lse3[b:b + 1, h0 * group:h1 * group].copy_(ls, non_blocking=True)
                if lmap is not None:
                    lmap[b:b + 1, h0 * group:h1 * group].copy_(res.plan.level_map, non_blocking=True)
                    res.plan.level_map.record_stream(s_out)
                freed = torch.cuda.Event()
                freed.record(s_out)
                sl["free_out"] = freed
        cur.wait_stream(s_out)
        s_out.synchronize()
        tail = torch.cat([counts, skipped, bad]).cpu().tolist()
    if tail[-1]:
        raise ValidationError("[stage: input] Q, K or V contains NaN or Inf entries")
    tail = tail[:-1]
    return StagedResult(out=out4.reshape(lead + (rows, d)),
                        lse=lse3.reshape(lead + (rows,)), level_counts=[int(c) for c in tail[:-1]],
                        skipped=int(tail[-1]), level_map=lmap)

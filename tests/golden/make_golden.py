"""Generate the golden fixtures from the REAL reference implementation.

Run in the build container (the reference is importable only here):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
It imports `pyrattn` read-only, feeds it bf16-rounded seeded inputs, and stores inputs plus the
reference's outputs as small .npz files next to this script. tests/test_oracle_golden.py (CPU)
pins the oracle to these files; tests/test_gpu_golden.py (GPU) checks the kernels against them.
Nothing at GPU-test time reads /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import pyrattn as ref  # noqa: E402


def bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16) \
        .to(torch.float64).numpy()


def bits(x):
    """bf16 payload (uint16) of bf16-representable float64 values."""
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).view(torch.int16) \
        .numpy().view(np.uint16)


def qkv(seed, n, d, kind="gaussian"):
    if kind == "gaussian":
        rng = np.random.default_rng(seed)
        return [bf16(rng.standard_normal((n, d), dtype=np.float32)) for _ in range(3)]
    g = 1 << ((n.bit_length() - 1) // 2)
    data = ref.synthesize("correlated", n, d, seed, grid=(g, n // g))
    return [bf16(data[x]) for x in ("q", "k", "v")]


def case(name, n, d, bq, bk, H, *, seed, kind="gaussian", estimator="sampled-max", s_q=8,
         s_k=8, mask="threshold", thresholds=None, cutpoints=None, tau=None, sim=None,
         causal=False, stride=None, keep_pyramid=False, grid=None, unpermute=False):
    q, k, v = qkv(seed, n, d, kind)
    lay = ref.make_layout(n, d, bq, bk, H)
    q_in, k_in, v_in = q, k, v
    perm = None
    if grid is not None:  # pipeline.py:257-263
        perm = ref.hilbert_order(grid)
        q, k, v = (ref.apply_permutation(x, perm) for x in (q, k, v))
    pyr = ref.build_pyramid(k, v, lay)
    if estimator == "antidiagonal":
        scores = ref.importance_antidiagonal(q, k, lay, stride)
    else:
        scores = ref.importance_sampled(q, k, lay, ref.SamplerConfig(s_q, s_k, 0),
                                        reducer="max" if estimator == "sampled-max" else "mean")
    if mask == "threshold":
        m = ref.assign_threshold(scores, ref.LevelThresholds(thresholds))
    elif mask == "binary":
        m = ref.binary_mask(scores, tau)
    else:
        pts = ref.QuantileCutpoints(cutpoints) if mask == "quantile" else ref.PRESET_CUTPOINTS[mask]
        m = ref.assign_quantile(scores, pts)
    caps = None
    if sim is not None:
        caps = ref.level_cap_from_similarity(pyr, ref.SimThresholds(sim))
        m = ref.combine_mask(m, caps)
    if causal:
        m = ref.causal_premask(m, lay)
    att = ref.psa_streaming(q, pyr, m, causal=causal)
    out, lse = att.out, att.row_log_normalizers
    if perm is not None and unpermute:  # pipeline.py:312-313 (lse follows out's row order)
        inv = ref.invert_permutation(perm)
        out = ref.apply_permutation(out, inv)
        lse = lse[inv.order]
    rep = ref.sparsity_report(m, levels=H)
    levels_k = [np.concatenate([pyr.k(j, h) for j in range(lay.n_k)]) for h in range(1, H + 1)]
    levels_v = [np.concatenate([pyr.v(j, h) for j in range(lay.n_k)]) for h in range(1, H + 1)]
    payload = dict(
        q=bits(q_in), k=bits(k_in), v=bits(v_in),
        layout=np.array([n, d, bq, bk, H]), scores=scores, mask=m,
        caps=caps if caps is not None else np.zeros(0, np.int64),
        out=out, lse=lse, skipped=np.array(att.skipped_rows),
        level_counts=np.array(rep.level_counts), rho_bar=np.array(rep.rho_bar),
        kv_coverage=np.array(rep.kv_coverage),
        config=np.array(repr(dict(estimator=estimator, s_q=s_q, s_k=s_k, seed=0, mask=mask,
                                  thresholds=thresholds, cutpoints=cutpoints, tau=tau,
                                  sim_thresholds=sim, causal=causal, stride=stride, grid=grid,
                                  unpermute=unpermute))),
    )
    for h in range(2, H + 1 if keep_pyramid else 2):
        payload[f"k_level{h}"] = levels_k[h - 1]
        payload[f"v_level{h}"] = levels_v[h - 1]
    np.savez_compressed(HERE / f"{name}.npz", **payload)
    print(name, "rho", rep.rho_bar, "skipped", att.skipped_rows)


TAUS = (0.164713, 0.282366, 0.376488, 0.95)

def hilbert_fixture():
    grids = [(4, 4), (8, 2), (2, 16), (16, 16), (64, 32), (3, 5, 6), (2, 3, 4), (5, 7, 9),
             (1, 8, 8), (21, 45, 80)]
    payload = {f"g{i}": np.array(g) for i, g in enumerate(grids)}
    payload.update({f"o{i}": ref.hilbert_order(g).order for i, g in enumerate(grids)})
    np.savez_compressed(HERE / "hilbert_orders.npz", **payload)


def schedule_fixture():
    """build_schedule / utilization of the reference (scheduler.py:71-126, 272-282)."""
    rng = np.random.default_rng(21)
    payload = {}
    cases = [  # (n, b_q, b_k, levels, tile_len, merge)
        (768, 64, 64, 4, 128, True), (768, 64, 64, 4, 128, False),
        (960, 120, 120, 4, 50, True), (960, 120, 120, 4, 50, False),
        (512, 128, 32, 3, 7, True), (256, 64, 64, 4, 64, True)]
    for c, (n, bq, bk, H, tile_len, merge) in enumerate(cases):
        lay = ref.make_layout(n, 64, bq, bk, H)
        m = rng.integers(0, H + 1, size=(lay.n_q, lay.n_k))
        sch = ref.build_schedule(m, lay, tile_len, merge=merge)
        rows = [(t.query_block, s.kv_block, s.level, s.row_start, s.row_stop, ti)
                for ti, t in enumerate(sch.tiles) for s in t.segments]
        u = ref.utilization(sch)
        payload[f"mask{c}"] = m
        payload[f"layout{c}"] = np.array([n, 64, bq, bk, H])
        payload[f"opts{c}"] = np.array([tile_len, int(merge)])
        payload[f"segs{c}"] = np.array(rows, dtype=np.int64).reshape(-1, 6)
        payload[f"util{c}"] = np.array([u.tiles, u.useful_rows, u.capacity, u.utilization])
    np.savez_compressed(HERE / "schedules.npz", **payload)


def pipeline_report_fixture():
    """run_pipeline report of the reference on 2 heads (pipeline.py:333-397)."""
    import json
    rng = np.random.default_rng(31)
    q, k, v = (bf16(rng.standard_normal((2, 1024, 64), dtype=np.float32)) for _ in range(3))
    cfg = ref.RunConfig.from_dict(dict(n=1024, d=64, b_q=64, b_k=64, levels=4,
                                       estimator="sampled-max", s_q=8, s_k=8, seed=0,
                                       mask="threshold", thresholds=list(TAUS), tile_len=128,
                                       num_steps=4, dense_prefix=0.25))
    res = ref.run_pipeline(cfg, q, k, v)
    rep = dict(res.report)
    rep.pop("wall_time_s")
    np.savez_compressed(HERE / "pipeline_report.npz", q=bits(q), k=bits(k), v=bits(v),
                        out=res.output, report=np.array(json.dumps(rep, sort_keys=True)))


def psat_fixture():
    """PSAT files written by the reference (tensorfile.py:28-41): bytes and the arrays read back."""
    import tempfile
    rng = np.random.default_rng(41)
    arrays = [rng.standard_normal(7), rng.standard_normal((3, 5)) * 1e3,
              rng.standard_normal((2, 4, 3)), np.array([[1.0, -0.0], [1e-40, 3.0e38]])]
    payload = {}
    with tempfile.TemporaryDirectory() as td:
        for i, a in enumerate(arrays):
            path = Path(td) / f"t{i}.psat"
            ref.write_tensor(path, a)
            payload[f"in{i}"] = a
            payload[f"bytes{i}"] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
            payload[f"read{i}"] = ref.read_tensor(path)
    np.savez_compressed(HERE / "psat_files.npz", **payload)


if __name__ == "__main__":
    psat_fixture()
    pipeline_report_fixture()
    hilbert_fixture()
    schedule_fixture()
    case("cfg1_small", 1024, 64, 64, 64, 4, seed=1, thresholds=TAUS, keep_pyramid=True)
    case("wan_b120", 960, 128, 120, 120, 4, seed=2, thresholds=(0.1634, 0.2803, 0.3738, 0.95),
         keep_pyramid=True)
    case("quantile_psa3", 512, 128, 64, 64, 4, seed=3, mask="psa-3")
    case("binary", 1024, 64, 64, 64, 1, seed=4, mask="binary", tau=0.6)
    case("simcap_corr", 1024, 64, 64, 64, 4, seed=5, kind="correlated", thresholds=TAUS,
         sim=(0.7, 0.65, 0.6))
    case("causal", 512, 128, 64, 64, 4, seed=6, thresholds=TAUS, causal=True)
    case("mean_reducer", 1024, 64, 64, 32, 3, seed=7, estimator="sampled-mean", s_q=5, s_k=7,
         thresholds=(0.3, 0.6, 0.9))
    case("antidiag", 1024, 64, 64, 64, 4, seed=8, estimator="antidiagonal", stride=8,
         thresholds=TAUS)
    case("dropped_rows", 512, 64, 64, 64, 2, seed=9, thresholds=(0.02, 0.05))
    # cfg4-style (Qwen prefill): antidiagonal stride 8 + similarity cap + causal pre-pass
    case("antidiag_causal_qwen", 1024, 128, 64, 64, 4, seed=10, estimator="antidiagonal",
         stride=8, thresholds=TAUS, sim=(0.75, 0.70, 0.70), causal=True)
    case("antidiag_stride4_b120", 960, 128, 120, 120, 4, seed=11, estimator="antidiagonal",
         stride=4, thresholds=(0.1634, 0.2803, 0.3738, 0.95))
    # space-filling-curve token order (pipeline.py:257-263, 312-313): 2D Hilbert and 3D serpentine
    case("hilbert2d_corr", 1024, 64, 64, 64, 4, seed=13, kind="correlated", thresholds=TAUS,
         grid=(32, 32), unpermute=True)
    case("hilbert3d_permuted_out", 960, 64, 64, 64, 4, seed=14, thresholds=TAUS, grid=(6, 10, 16))
    # stride does not divide q_block: residue classes of unequal size
    case("antidiag_ragged", 960, 64, 60, 48, 4, seed=12, estimator="antidiagonal", stride=8,
         thresholds=TAUS)

"""Parity at the benchmarked shapes (VERDICT r01 "next" #1).

The GPU runs the fused forward over every head of the bench workload (bench.py CONFIGS, the same
seeded torch.Generator inputs as the bench); the CPU oracle re-derives, for a subset of heads,

  level map          == (pkg/src/pyrattn/mask.py:128-151, importance.py:52-85 / :97-132,
                        mask.py:198-234 cap, mask.py:324-349 causal pre-pass)
  selected blocks    == : the plan rows (level-major, ascending j) and their slot-row totals
  O / lse            on 16 query blocks per head spread over the sequence (attention.py:120-168
                        materialized per query block, the bf16 pyramid the kernel consumes):
                        rel-L2 <= 5e-3, max-abs <= 1e-2 * max|ref|, |lse - ref| <= 1e-3

cfg2: all 12 heads. cfg3: 4 heads (assign_levels_kernel<5,5>, n_k = 630, ~120 KV tiles per
unit). cfg4: 4 query heads spanning the kv-head 0 / 1 GQA boundary (antidiagonal stride 8,
similarity cap, causal).
"""

import numpy as np
import pytest
import torch

from helpers import bf16_round, rel_l2
from oracle import psa_oracle as orc

pytestmark = pytest.mark.gpu

O_BLOCKS = 16


def _bench():
    import bench
    return bench


def _plan_rows_from_mask(m, lay):
    """Expected plan rows of one head: level-major, ascending j; Σ power-of-two slot rows."""
    rows, totals = [], []
    for i in range(m.shape[0]):
        ent, tot = [], 0
        for h in range(1, lay.levels + 1):
            L = lay.pooled_len(h)
            slot = max(8, 1 << (L - 1).bit_length())
            js = np.nonzero(m[i] == h)[0]
            ent += [int(j) | (h << 12) for j in js]
            tot += slot * js.size
        rows.append(ent)
        totals.append(tot)
    return rows, totals


def _run(cfg_name, check_heads):
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.pipeline import psa_forward_4d

    bench = _bench()
    cfg = bench.CONFIGS[cfg_name]
    Hq, Hkv = cfg["Hq"], cfg["Hkv"]
    group = Hq // Hkv
    q, k, v = bench.make_inputs(cfg, list(range(Hq)), list(range(Hkv)), torch.device("cuda"))
    rc = bench.run_config(cfg)
    res = psa_forward_4d(q, k, v, rc)
    torch.cuda.synchronize()
    lay = orc.Layout(cfg["N"], cfg["d"], cfg["b_q"], cfg["b_k"], cfg["levels"])
    lm = res.plan.level_map[0].cpu().numpy()
    csr = res.plan.csr.to(torch.int32).bitwise_and(0xFFFF).cpu().numpy()
    info = res.plan.info.cpu().numpy()
    out = res.out[0]
    lse = res.lse[0]
    blocks = np.unique(np.linspace(0, lay.n_q - 1, O_BLOCKS).round().astype(int))
    stats = {"mismatch": 0, "rel": 0.0, "mabs": 0.0, "lse": 0.0}
    for h in check_heads:
        hk = h // group
        qh = q[0, h].to(torch.float64).cpu().numpy()
        kh = k[0, hk].to(torch.float64).cpu().numpy()
        vh = v[0, hk].to(torch.float64).cpu().numpy()
        r = orc.run_head(qh, kh, vh, lay, estimator=cfg["estimator"], s_q=8, s_k=8, seed=0,
                         stride=cfg["stride"], mask="threshold", thresholds=cfg["taus"],
                         sim_thresholds=cfg["sim"], causal=cfg["causal"],
                         executor="materialized", rows_of=[])
        m = r["mask"]
        mism = int((lm[h] != m).sum())
        stats["mismatch"] += mism
        assert mism == 0, f"{cfg_name} head {h}: {mism} level-map mismatches"
        rows, totals = _plan_rows_from_mask(m, lay)
        base = h * lay.n_q
        for i in range(lay.n_q):
            n_ent = int(info[base + i, 0])
            assert n_ent == len(rows[i]), (cfg_name, h, i)
            assert int(info[base + i, 1]) == totals[i], (cfg_name, h, i)
            assert csr[base + i, :n_ent].tolist() == rows[i], (cfg_name, h, i)
        kl, vl = r["pyramid"]
        kl = [bf16_round(x) for x in kl]
        vl = [bf16_round(x) for x in vl]
        ref_o, ref_l, _ = orc.psa_materialized(qh, kl, vl, m, lay, cfg["causal"], rows_of=blocks)
        sel = np.concatenate([np.arange(i * lay.q_block, (i + 1) * lay.q_block) for i in blocks])
        got_o = out[h][torch.from_numpy(sel).cuda()].double().cpu().numpy()
        got_l = lse[h][torch.from_numpy(sel).cuda()].double().cpu().numpy()
        ro, rl = ref_o[sel], ref_l[sel]
        e_rel = rel_l2(got_o, ro)
        e_abs = float(np.abs(got_o - ro).max())
        assert e_rel <= 5e-3, (cfg_name, h, e_rel)
        assert e_abs <= 1e-2 * float(np.abs(ro).max()), (cfg_name, h, e_abs)
        fin = np.isfinite(rl)
        assert np.array_equal(np.isfinite(got_l), fin)
        e_l = float(np.abs(got_l[fin] - rl[fin]).max()) if fin.any() else 0.0
        assert e_l <= 1e-3, (cfg_name, h, e_l)
        stats["rel"] = max(stats["rel"], e_rel)
        stats["mabs"] = max(stats["mabs"], e_abs / float(np.abs(ro).max()))
        stats["lse"] = max(stats["lse"], e_l)
    total = [int(c) for c in res.plan.level_counts.cpu().tolist()]
    print(f"{cfg_name}: heads {list(check_heads)} level-map mismatches {stats['mismatch']}, "
          f"worst O rel-L2 {stats['rel']:.2e}, max-abs/max|ref| {stats['mabs']:.2e}, "
          f"lse {stats['lse']:.2e}; rho_bar {psa.report_from_counts(total, sum(total)).rho_bar:.4f}")
    return stats


def test_fullshape_cfg2_all_heads():
    _run("cfg2", range(12))


def test_fullshape_cfg3_four_heads():
    _run("cfg3", (0, 13, 26, 39))


def test_fullshape_cfg4_gqa_boundary():
    _run("cfg4", (5, 6, 7, 8))

"""Bisect the threshold scale alpha of T = (alpha*0.35, alpha*0.6, alpha*0.8, 0.95) to a target
rho_bar on the CPU oracle, as the reference's acceptance test does
(pkg/tests/test_acceptance.py:130-176, _bisect_to_budget). rho_bar is the reference's
sparsity_report over all n_q x n_k entries (mask.py:278-321), after the similarity cap and the
causal pre-pass when the config has them.

    python scripts/calibrate_budget.py --config cfg4 --heads 4 --target 0.20
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--target", type=float, default=0.20)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--scale-all", action="store_true",
                    help="scale all four thresholds (alpha*(0.35, 0.6, 0.8, 0.95)); needed when the "
                         "similarity cap holds pooled levels down, so only dropping blocks moves "
                         "the budget")
    args = ap.parse_args()
    import bench
    from oracle import psa_oracle as orc
    cfg = bench.CONFIGS[args.config]
    lay = orc.Layout(cfg["N"], cfg["d"], cfg["b_q"], cfg["b_k"], cfg["levels"])
    group = cfg["Hq"] // cfg["Hkv"]
    heads = [h * cfg["Hq"] // args.heads for h in range(args.heads)]  # spread over kv groups
    rng = np.random.default_rng(2026)
    per_head = []
    for h in heads:
        import torch
        q, k = (torch.from_numpy(rng.standard_normal((cfg["N"], cfg["d"]), dtype=np.float32))
                .to(torch.bfloat16).to(torch.float64).numpy() for _ in range(2))
        if cfg["estimator"] == "antidiagonal":
            s = orc.importance_antidiagonal(q, k, lay, cfg["stride"])
        else:
            s = orc.importance_sampled(q, k, lay, 8, 8, 0)
        caps = orc.level_caps(k, lay, cfg["sim"]) if cfg["sim"] else None
        per_head.append((s, caps))
        print(f"head {h} (kv {h // group}) importance done", flush=True)

    def rho(alpha):
        taus = (alpha * 0.35, alpha * 0.6, alpha * 0.8, alpha * 0.95 if args.scale_all else 0.95)
        counts = np.zeros(lay.levels + 1, dtype=np.int64)
        for s, caps in per_head:
            m = orc.assign_threshold(s, taus)
            if caps is not None:
                m = orc.combine_mask(m, caps)
            if cfg["causal"]:
                m = orc.causal_premask(m, lay)
            counts += np.bincount(m.reshape(-1), minlength=lay.levels + 1)
        return orc.report_from_counts(counts.tolist(), int(counts.sum()))["rho_bar"]

    lo, hi, best = 0.0, 1.0, None
    for _ in range(args.iters):
        mid = 0.5 * (lo + hi)
        r = rho(mid)
        if best is None or abs(r - args.target) < abs(best[1] - args.target):
            best = (mid, r)
        lo, hi = (mid, hi) if r < args.target else (lo, mid)
    a = best[0]
    last = a * 0.95 if args.scale_all else 0.95
    print(f"alpha={a:.6f} rho_bar={best[1]:.5f} "
          f"taus={[round(a * 0.35, 6), round(a * 0.6, 6), round(a * 0.8, 6), round(last, 6)]}")


if __name__ == "__main__":
    main()

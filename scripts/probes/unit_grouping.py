"""dK/dV row packing: live-row fraction of different block groupings per level (cfg3 level map)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_04025_b200 as psa  # noqa: E402

cfg = bench.CONFIGS["cfg3"]
dev = torch.device("cuda:0")
q, k, v = bench.make_inputs(cfg, list(range(cfg["Hq"])), list(range(cfg["Hkv"])), dev)
res = psa.psa_forward_4d(q, k, v, bench.run_config(cfg))
lm = res.plan.level_map  # [B, H, n_q, n_k]
nk = lm.shape[-1]
for h in range(2, cfg["levels"] + 1):
    f = 1 << (h - 1)
    hit = (lm == h)
    for name, stride in [("neighbours", 1), ("stride 2", 2), ("stride 8", 8), ("stride nk/f", nk // f)]:
        m = (nk // (f * stride)) * f * stride if stride > 1 else (nk // f) * f
        x = hit[..., :m]
        if stride == 1:
            g = x.reshape(*x.shape[:-1], -1, f)
        else:
            g = x.reshape(*x.shape[:-1], -1, f, stride).transpose(-1, -2).reshape(*x.shape[:-1], -1, f)
        ent = int(g.any(-1).sum())
        live = int(g.sum())
        print(f"level {h} {name:12s}: entries {ent:9d} live {live:9d} fraction {live / max(ent * f, 1):.3f}")
    # best case: per query row, selected blocks sorted and packed (greedy lower bound on entries)
    per_row = hit.sum(-1)
    ent_lb = int(((per_row + f - 1) // f).sum())
    print(f"level {h} lower bound (perfect packing per query block): entries {ent_lb}")

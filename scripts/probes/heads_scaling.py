"""Per-stage time of the cfg3 forward on H of the 40 heads (what one rank runs at N = 40 / H GPUs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2512_04025_b200.attention import attention_forward  # noqa: E402
from paper_2512_04025_b200.importance import importance_scores  # noqa: E402
from paper_2512_04025_b200.layout import LevelThresholds, SamplerConfig  # noqa: E402
from paper_2512_04025_b200.mask import assign_levels_device  # noqa: E402
from paper_2512_04025_b200.pyramid import build_pyramid  # noqa: E402

cfg = bench.CONFIGS["cfg3"]
dev = torch.device("cuda:0")
lay = bench.run_config(cfg).layout()
for H in (40, 20, 10, 5):
    q, k, v = bench.make_inputs(cfg, list(range(H)), list(range(H)), dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def step(rec):
        if rec: ev[0].record()
        pyr = build_pyramid(k, v, lay)
        if rec: ev[1].record()
        sc = importance_scores(q, k, lay, SamplerConfig(8, 8, 0), "max")
        if rec: ev[2].record()
        plan = assign_levels_device(sc, mode="threshold", rule=LevelThresholds(cfg["taus"]),
                                    levels=lay.levels, b_q=lay.q_block, b_k=lay.k_block,
                                    hkv=H, caps=None, causal=False)
        if rec: ev[3].record()
        attention_forward(q, pyr, plan, False)
        if rec: ev[4].record()

    for _ in range(3):
        step(False)
    tot = [0.0] * 4
    for _ in range(5):
        step(True)
        torch.cuda.synchronize()
        for i in range(4):
            tot[i] += ev[i].elapsed_time(ev[i + 1]) / 5
    print(f"H={H:2d} per-head ms: " + " ".join(f"{n}={t / H:.4f}" for n, t in
                                             zip(("pyr", "imp", "assign", "attn"), tot)),
          f"total/head {sum(tot) / H:.4f}")
    del q, k, v

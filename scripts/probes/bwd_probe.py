"""Backward: gradient errors vs the fp64 oracle (small case) and device time at cfg3 shape."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import paper_2512_04025_b200 as psa  # noqa: E402
from helpers import gaussian_qkv, rel_l2, to_dev  # noqa: E402
from paper_2512_04025_b200.attention import attention_backward  # noqa: E402
from test_gpu_backward import _oracle  # noqa: E402

for (n, d, bq, bk, hq, hkv, causal) in [(1024, 64, 64, 64, 2, 2, False), (960, 128, 120, 120, 2, 1, False),
                                         (1024, 128, 128, 64, 4, 2, True)]:
    q, k, v = gaussian_qkv(61, hq, n, d, hkv)
    g = np.random.default_rng(62).standard_normal((hq, n, d))
    cfg = psa.RunConfig.from_dict(dict(n=n, d=d, b_q=bq, b_k=bk, levels=4, estimator="sampled-max",
                                       s_q=8, s_k=8, seed=0, mask="threshold",
                                       thresholds=[0.25, 0.45, 0.6, 0.9], tile_len=128, causal=causal))
    q4, k4, v4 = (to_dev(x)[None] for x in (q, k, v))
    res = psa.psa_forward_4d(q4, k4, v4, cfg)
    lm = res.plan.level_map[0].cpu().numpy()
    dq, dk, dv = attention_backward(q4, res.pyramid, res.plan, causal, res.out, res.lse, to_dev(g)[None])
    qt, kt, vt = (torch.from_numpy(x).requires_grad_(True) for x in (q, k, v))
    out = _oracle(qt, kt, vt, lm, bq, bk, causal)
    (out * torch.from_numpy(g)).sum().backward()
    errs = [rel_l2(m[0].float().cpu().numpy(), r.numpy()) for m, r in ((dq, qt.grad), (dk, kt.grad), (dv, vt.grad))]
    print("case", (n, d, bq, bk, hq, hkv, causal), "levels", np.bincount(lm.ravel(), minlength=5), "rel err dq dk dv", [f"{e:.2e}" for e in errs])

cfg = bench.CONFIGS["cfg3"]
dev = torch.device("cuda:0")
q, k, v = bench.make_inputs(cfg, list(range(cfg["Hq"])), list(range(cfg["Hkv"])), dev)
rc = bench.run_config(cfg)
res = psa.psa_forward_4d(q, k, v, rc)
g = torch.randn_like(q)
for _ in range(2):
    attention_backward(q, res.pyramid, res.plan, False, res.out, res.lse, g)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    attention_backward(q, res.pyramid, res.plan, False, res.out, res.lse, g)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
counts = res.plan.level_counts.cpu().tolist()
sel_blocks = sum(counts[1:])
flops = 2.5 * 4 * cfg["d"] * sel_blocks * cfg["b_q"] * cfg["b_k"]  # expanded blocks: S, dP, dV, dK, dQ
print(f"cfg3 backward {ms:.2f} ms; selected blocks {sel_blocks}; {flops / ms / 1e9:.0f} TFLOP/s on expanded-block work")
alg = 2.5 * bench.flops_from_counts(counts, cfg, cfg["B"] * cfg["Hq"])  # pooled work: 5 GEMMs vs 2
print(f"cfg3 backward algorithmic work {alg / 1e12:.1f} TFLOP (2.5x the forward's): {alg / ms / 1e9:.0f} TFLOP/s")

# per-kernel device times (CUPTI) of the same calls
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        attention_backward(q, res.pyramid, res.plan, False, res.out, res.lse, g)
    torch.cuda.synchronize()
for ev in prof.key_averages():
    if ev.device_type.name == "CUDA" and ev.count:
        print(f"  {ev.key[:60]:60s} x{ev.count:3d} {ev.device_time_total / ev.count / 1e3:9.3f} ms")

# dK/dV row packing: MMA rows that carry a selected block, per level (live rows / tile rows)
lm = res.plan.level_map.to(torch.int16)
nk = lm.shape[-1]
for h in range(1, cfg["levels"] + 1):
    f = 1 << (h - 1)
    pad = (-nk) % f
    hit = torch.nn.functional.pad((lm == h).to(torch.int16), (0, pad)).view(*lm.shape[:-1], -1, f)
    ent = int(hit.any(-1).sum())
    live = int(hit.sum())
    eff = live / max(ent * f, 1)
    print(f"  level {h}: entries {ent:9d}  selected blocks {live:9d}  live-row fraction {eff:.3f}")

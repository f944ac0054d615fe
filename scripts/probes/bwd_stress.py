"""Repeat the backward many times (hang / race check) at the cfg3 shape and on small shapes."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_04025_b200 as psa  # noqa: E402
from paper_2512_04025_b200.attention import attention_backward  # noqa: E402

cfg = bench.CONFIGS["cfg3"]
dev = torch.device("cuda:0")
q, k, v = bench.make_inputs(cfg, list(range(cfg["Hq"])), list(range(cfg["Hkv"])), dev)
res = psa.psa_forward_4d(q, k, v, bench.run_config(cfg))
g = torch.randn_like(q)
ref = attention_backward(q, res.pyramid, res.plan, False, res.out, res.lse, g)
t0 = time.time()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for it in range(n):
    out = attention_backward(q, res.pyramid, res.plan, False, res.out, res.lse, g)
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(out, ref))
    if not same:
        print("iteration", it, "differs from the first run")
print(f"{n} cfg3 backward runs in {time.time() - t0:.1f} s, deterministic")

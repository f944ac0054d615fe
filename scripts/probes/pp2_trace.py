"""Per-tile event trace of psa_attn_pp2_kernel. Apply scripts/probes/pp2_trace.patch to
psa_attention.cu as of commit 4e7e050 (`git checkout 4e7e050 -- paper_2512_04025_b200/csrc`) first (adds
the PSA_PP2_VAR=4|5 builds that record clock64 stamps for 8 CTAs mid-grid): MMA S/PV issue, lane
S-ready / wait-start / P-done, K TMA issue, K/V ready at the MMA warp. cfg3 shapes."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2512_04025_b200 import _lib  # noqa: E402
from paper_2512_04025_b200.attention import attention_forward  # noqa: E402
from paper_2512_04025_b200.importance import importance_scores  # noqa: E402
from paper_2512_04025_b200.layout import LevelThresholds, SamplerConfig  # noqa: E402
from paper_2512_04025_b200.mask import assign_levels_device  # noqa: E402
from paper_2512_04025_b200.pyramid import build_pyramid  # noqa: E402

cfg = bench.CONFIGS["cfg3"]
dev = torch.device("cuda:0")
q, k, v = bench.make_inputs(cfg, list(range(cfg["Hq"])), list(range(cfg["Hkv"])), dev)
lay = bench.run_config(cfg).layout()
pyr = build_pyramid(k, v, lay)
scores = importance_scores(q, k, lay, SamplerConfig(8, 8, 0), "max")
plan = assign_levels_device(scores, mode="threshold", rule=LevelThresholds(cfg["taus"]),
                            levels=lay.levels, b_q=lay.q_block, b_k=lay.k_block, hkv=k.shape[1],
                            caps=None, causal=False)
for _ in range(3):
    attention_forward(q, pyr, plan, False)
torch.cuda.synchronize()
buf = np.zeros((8, 10, 256), dtype=np.int64)
lib = _lib.load()
lib.psa_debug_pp2_trace.argtypes = [ctypes.c_void_p]
assert lib.psa_debug_pp2_trace(buf.ctypes.data) == 0
tiles = plan.info[:, 1].cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/pp2_trace_{os.environ.get('PSA_PP2_VAR', '0')}.npz", trace=buf,
         rows=np.array([tiles[1234 + 3000 * s] for s in range(8)]))
print("ok")

"""Per-tile clock64 trace of psa_attn_pp2_kernel at cfg3 (8 CTAs mid-grid) from the instrumented
build (scripts/probes/build_trace_lib.sh; run with PSA_LIB_PATH=scripts/probes/libpsa_trace.so).
Events per tile t: 0 lane wait start, 1 S ready, 2 LDTM done, 3 max done, 4 exps/sums done,
5 P stored + arrived, 6 S(t) issued by the MMA warp, 7 PV(t) issued. Prints per-phase medians."""
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

cfg = bench.CONFIGS[os.environ.get("CFG", "cfg3")]
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
buf = np.zeros((8, 16, 256), dtype=np.int64)
lib = _lib.load()
lib.psa_debug_pp2_trace.argtypes = [ctypes.c_void_p]
assert lib.psa_debug_pp2_trace(buf.ctypes.data) == 0
rows = plan.info[:, 1].cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/pp2_trace2.npz", trace=buf, rows=np.array([rows[1234 + 3000 * s] for s in range(8)]))
dump = os.environ.get("DUMP")
names = ["wait->S ready", "S ready->LDTM done", "LDTM->max done", "max->exps done", "exps->P arrived"]
for s in range(8):
    T = (int(rows[1234 + 3000 * s]) + 127) // 128
    tr = buf[s][:, :min(T, 256)]
    t0 = tr[0, 0]
    mid = slice(4, min(T, 256) - 4)
    ph = [np.median(tr[e + 1, mid] - tr[e, mid]) for e in range(5)]
    period = np.median(np.diff(tr[5, mid][::2]))
    s_issue_to_ready = np.median(tr[1, mid] - tr[6, mid])
    pv_issue_after_p = np.median(tr[7, mid] - tr[5, mid])
    idx = np.arange(6, min(T, 256) - 4)
    kland = np.median(tr[9, idx] - tr[8, idx])
    cur = np.median(tr[11, idx] - tr[10, idx])
    k_after = np.median(tr[8, idx] - tr[1, idx - 2])
    print(f"   MMA: enter issue_s(t+2) - P(t) {np.median(tr[10, idx + 2] - tr[5, idx]):.0f} | k_full(t+2) pass - P(t) {np.median(tr[11, idx + 2] - tr[5, idx]):.0f} | S(t+2) issued - P(t) {np.median(tr[6, idx + 2] - tr[5, idx]):.0f} | enter pv(t) - P(t) {np.median(tr[13, idx] - tr[5, idx]):.0f} | v_full(t) pass - P(t) {np.median(tr[12, idx] - tr[5, idx]):.0f} | K(t+2) landed - P(t) {np.median(tr[9, idx + 2] - tr[5, idx]):.0f}")
    print(f"   K TMA issue->landed {kland:.0f} | MMA cursor {cur:.0f} | K(t) TMA issue - S(t-2) ready {k_after:.0f}")
    print(f"cta {s}: T={T} lane period {period:.0f} cyc | " + " | ".join(f"{n} {v:.0f}" for n, v in zip(names, ph))
          + f" | S issue->ready {s_issue_to_ready:.0f} | P->PV issue {pv_issue_after_p:.0f}")

if dump:
    s = 2
    t0 = buf[s, 5, 40]
    print("t  Kloop  kempty  Kissue  TMAdone in_s  kfull  Sissd  Srdy  Pdone  in_pv  vfull  PVissd")
    for t in range(40, 50):
        e = buf[s, :, t] - t0
        print(t, e[15], e[14], e[8], e[9], e[10], e[11], e[6], e[1], e[5], e[13], e[12], e[7])

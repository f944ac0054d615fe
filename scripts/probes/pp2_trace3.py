"""Per-tile clock64 trace of psa_attn_pp2_kernel (8 CTAs spaced through the grid) from the
instrumented build: scripts/probes/build_trace_lib.sh, then run with
PSA_LIB_PATH=scripts/probes/libpsa_trace.so. Events per KV tile t (psa_attention.cu, PSA_TRACE):
0 lane (t&1) waits for S(t), 1 S(t) ready, 2 max done, 3 exps done, 4 P(t) released,
5 S(t) issued, 6 PV(t) issued, 7 MMA warp waits for P(t), 8 K(t) TMA issued, 9 V(t) TMA issued,
10 segments of K tile t, 11/12/13 the MMA warp sees K(t) full / s_free / aug_full.
Prints steady-state per-phase medians and a timeline of one CTA."""
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
heads = int(os.environ.get("HEADS", cfg["Hq"]))
q, k, v = bench.make_inputs(cfg, list(range(heads)), list(range(heads)), dev)
lay = bench.run_config(cfg).layout()
pyr = build_pyramid(k, v, lay)
scores = importance_scores(q, k, lay, SamplerConfig(8, 8, 0), "max")
plan = assign_levels_device(scores, mode="threshold", rule=LevelThresholds(cfg["taus"]),
                            levels=lay.levels, b_q=lay.q_block, b_k=lay.k_block, hkv=k.shape[1],
                            caps=None, causal=False)
for _ in range(3):
    attention_forward(q, pyr, plan, False)
torch.cuda.synchronize()
buf = np.zeros((8, 14, 256), dtype=np.int64)
lib = _lib.load()
lib.psa_debug_pp2_trace.argtypes = [ctypes.c_void_p]
assert lib.psa_debug_pp2_trace(buf.ctypes.data) == 0
os.makedirs("gpurun_out", exist_ok=True)
np.save(os.environ.get("TRACE_OUT", "gpurun_out/pp2_trace3.npy"), buf)

ph = {k_: [] for k_ in ("S wait", "ldtm+max", "exp", "store+release", "S issue->ready",
                        "P ready->PV issue", "MMA waits P", "lane period (2 tiles)",
                        "exp overlap with other lane", "K issue->S issue")}
for s in range(8):
    tr = buf[s]
    T = int((tr[1] > 0).sum())
    for t in range(4, T - 4):
        e = tr[:, t]
        ph["S wait"].append(e[1] - e[0])
        ph["ldtm+max"].append(e[2] - e[1])
        ph["exp"].append(e[3] - e[2])
        ph["store+release"].append(e[4] - e[3])
        ph["S issue->ready"].append(e[1] - e[5])
        ph["P ready->PV issue"].append(e[6] - e[4])
        ph["MMA waits P"].append(max(0, e[4] - e[7]))
        ph["lane period (2 tiles)"].append(tr[1, t + 2] - e[1])
        o = tr[:, t + 1]  # other lane's neighbouring tile
        ph["exp overlap with other lane"].append(
            max(0, min(e[3], o[3]) - max(e[2], o[2])) / max(1, e[3] - e[2]))
        ph["K issue->S issue"].append(e[5] - e[8])
# K latency (TMA issue -> the MMA warp sees the stage full) against the tile's segment count
lat = {}
for s in range(8):
    tr = buf[s]
    T = int((tr[1] > 0).sum())
    for t in range(2, T):
        lat.setdefault(int(tr[10, t]), []).append(tr[11, t] - tr[8, t])
print("K(t) issue -> full, by segments in the tile:")
for nseg in sorted(lat):
    print(f"  {nseg:2d} segments: n={len(lat[nseg]):4d} median {np.median(lat[nseg]):7.0f}")
ph["MMA: K full -> s_free"] = []
ph["MMA: s_free -> aug_full"] = []
for s in range(8):
    tr = buf[s]
    T = int((tr[1] > 0).sum())
    for t in range(4, T - 4):
        ph["MMA: K full -> s_free"].append(tr[12, t] - tr[11, t])
        ph["MMA: s_free -> aug_full"].append(tr[13, t] - tr[12, t])
for k_, v_ in ph.items():
    if v_:
        print(f"{k_:30s} median {np.median(v_):9.1f}   p10 {np.percentile(v_, 10):9.1f}   "
              f"p90 {np.percentile(v_, 90):9.1f}")
tr = buf[3]
t0 = tr[5, 0]
print("\ntimeline CTA slot 3 (cycles from S(0) issue): t | Kiss Kfull Siss Sready maxdone expdone Prel Viss PVwait PViss")
for t in range(8, 20):
    e = tr[:, t] - t0
    print(f"{t:3d} L{t & 1} | {e[8]:8d} {e[11]:8d} {e[5]:8d} {e[1]:8d} {e[2]:8d} {e[3]:8d} {e[4]:8d} {e[9]:8d} {e[7]:8d} {e[6]:8d}")
vk = []
for s in range(8):
    tr_ = buf[s]
    T = int((tr_[1] > 0).sum())
    for t in range(4, T - 4):
        vk.append((tr_[9, t], tr_[7, t], tr_[8, t + 1]))
vk = np.array(vk)
print("V(t) issue -> MMA reaches PV(t) (median):", np.median(vk[:, 1] - vk[:, 0]))

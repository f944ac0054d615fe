"""PSA forward benchmark (BASELINE.json metric: "PSA fwd ms & effective TFLOPS at Wan2.1-14B 720p
shape, 1/2/4/8 B200 vs CPU ref").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3]

A step is one full PSA forward (pyramid -> fp64 sampled importance -> Alg. 2 level map ->
multi-level tcgen05 attention) over every head of the workload, inputs resident in HBM.
Multi-GPU (torchrun): heads are sharded across ranks (no data-path collective), the timed region
is bracketed by barriers and the reported time is the max over ranks. rank 0 prints ONE JSON line.
--impl reference times the CPU oracle port of the reference path on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ALPHA = 0.4673  # threshold scale giving rho_bar ~= 0.20 at the Wan shapes
WAN_TAUS = (ALPHA * 0.35, ALPHA * 0.6, ALPHA * 0.8, 0.95)
# cfg4 (antidiagonal + similarity cap + causal): on synthetic Gaussian keys the cap holds every
# block at level 1 (adjacent keys are not similar), so only dropping blocks moves the budget; all
# four thresholds scale: alpha bisected on the CPU oracle to rho_bar = 0.20 over all n_q x n_k
# entries (scripts/calibrate_budget.py --config cfg4 --scale-all; test_acceptance.py:130-176)
CFG4_ALPHA = 0.431938
CFG4_TAUS = (CFG4_ALPHA * 0.35, CFG4_ALPHA * 0.6, CFG4_ALPHA * 0.8, CFG4_ALPHA * 0.95)

CONFIGS = {
    "cfg1": dict(desc="synthetic B=1 H=2 L=4096 d=64 (CPU-runnable case)", B=1, Hq=2, Hkv=2,
                 N=4096, d=64, b_q=64, b_k=64, levels=4,
                 taus=(0.164713, 0.282366, 0.376488, 0.95), causal=False),
    "cfg2": dict(desc="Wan2.1-1.3B 480p/81f: L=32760 H=12 d=128", B=1, Hq=12, Hkv=12, N=32760,
                 d=128, b_q=120, b_k=120, levels=4, taus=WAN_TAUS, causal=False),
    "cfg3": dict(desc="Wan2.1-14B 720p/81f: L=75600 H=40 d=128", B=1, Hq=40, Hkv=40, N=75600,
                 d=128, b_q=120, b_k=120, levels=4, taus=WAN_TAUS, causal=False),
    "cfg5": dict(desc="compute-budget sweep 10-50% at L=32760 H=12 d=128 vs dense and binary "
                      "(quantile cutpoints 0.6b,b,1.8b,1.8b -> rho_bar=b; binary = b at level 1)",
                 B=1, Hq=12, Hkv=12, N=32760, d=128, b_q=120, b_k=120, levels=4, taus=WAN_TAUS,
                 causal=False),
    "cfg4": dict(desc="Qwen2.5-VL-7B-style prefill: L=32768 Hq=28 Hkv=4 d=128 causal, "
                      "antidiagonal stride 8 + similarity cap (0.75,0.70,0.70)", B=1, Hq=28,
                 Hkv=4, N=32768, d=128, b_q=128, b_k=64, levels=4, taus=CFG4_TAUS, causal=True,
                 estimator="antidiagonal", stride=8, sim=(0.75, 0.70, 0.70)),
}
for _c in CONFIGS.values():
    _c.setdefault("estimator", "sampled-max")
    _c.setdefault("stride", None)
    _c.setdefault("sim", None)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled through NVML every ~2 ms by a background thread
    DURING the timed region (B200_PROFILING.md clocks line); short timed regions still get
    samples. Falls back to ``nvidia-smi -lms 50`` when NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.rows = []
        self._thread = None
        self._stop = None
        self._nvml = None

    def _sample(self):
        nv = self._nvml
        try:
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            pw = nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0
            self.rows.append((sm, self._max, pw, tuple(bool(rs & bt) for bt in self._bits)))
        except Exception:  # noqa: BLE001 - sampling must never kill the bench
            pass

    def _poll(self):
        while not self._stop.wait(self.period):
            self._sample()

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._bits = (nv.nvmlClocksEventReasonHwSlowdown,
                          nv.nvmlClocksEventReasonHwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwPowerCap)
            self._nvml = nv
        except Exception:  # noqa: BLE001
            self._nvml = None
        self._stop = threading.Event()
        if self._nvml is not None:  # one sample at entry, every ~2 ms after, one at exit
            self._sample()
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
        else:
            self._smi = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)
            self._sample()
            return
        self._smi.terminate()
        out, _ = self._smi.communicate(timeout=5)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(f[0]), float(f[1]), float(f[2]),
                                  tuple(x == "Active" for x in f[3:7])))
            except (ValueError, IndexError):
                pass

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[3][i]}),
                "power_w_max": max(r[2] for r in self.rows), "samples": len(self.rows),
                "sampler": "nvml 2 ms" if self._thread is not None else "nvidia-smi 50 ms"}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------------- workload
def make_inputs(cfg, heads, kv_heads, device, seed=0):
    """Synthetic N(0,1) bf16 Q/K/V generated per global head index (shard-invariant)."""
    import torch
    B, N, d = cfg["B"], cfg["N"], cfg["d"]
    out = []
    for name, hs in (("q", heads), ("k", kv_heads), ("v", kv_heads)):
        t = torch.empty(B, len(hs), N, d, dtype=torch.bfloat16, device=device)
        for bi in range(B):
            for li, h in enumerate(hs):
                g = torch.Generator(device=device)
                g.manual_seed(seed * 1_000_003 + {"q": 0, "k": 1, "v": 2}[name] * 10_007 + bi * 997 + h)
                t[bi, li] = torch.randn(N, d, generator=g, device=device, dtype=torch.float32)
        out.append(t)
    return out


def run_config(cfg):
    from paper_2512_04025_b200 import RunConfig
    return RunConfig.from_dict(dict(n=cfg["N"], d=cfg["d"], b_q=cfg["b_q"], b_k=cfg["b_k"],
                                    levels=cfg["levels"], estimator=cfg["estimator"], s_q=8, s_k=8,
                                    seed=0, stride=cfg["stride"], mask="threshold",
                                    thresholds=list(cfg["taus"]), sim_thresholds=cfg["sim"],
                                    tile_len=128, causal=cfg["causal"]))


def flops_from_counts(counts, cfg, heads=1):
    """Executed algorithmic FLOPs = 4*d*sum_h count_h * b_q * (b_k >> (h-1)),
    over ``heads`` (batch*q-head) units. Causal: the straddling level-1 pairs (always present
    after the causal pre-pass, mask.py:324-349) count only their visible (q, k) pairs."""
    d, bq, bk = cfg["d"], cfg["b_q"], cfg["b_k"]
    f = 4 * d * sum(int(c) * bq * (bk >> (h - 1)) for h, c in enumerate(counts) if h >= 1)
    if cfg["causal"]:
        f -= 4 * d * heads * _causal_hidden_pairs(cfg["N"], bq, bk)
    return f


def _causal_hidden_pairs(n, bq, bk):
    """Number of masked (q, k) pairs inside straddling level-1 block pairs of one head."""
    return _causal_hidden_pairs_blocks(n, bq, bk, range(n // bq))


def _causal_hidden_pairs_blocks(n, bq, bk, blocks):
    """Masked (q, k) pairs inside the straddling level-1 block pairs of the given query blocks."""
    hidden = 0
    for i in blocks:
        q_lo, q_hi = i * bq, i * bq + bq - 1
        for j in range(q_lo // bk, min(n // bk, q_hi // bk + 1)):
            k_lo = j * bk
            if k_lo + bk - 1 <= q_lo:
                continue  # fully visible
            for r in range(q_lo, q_hi + 1):
                vis = max(0, min(bk, r - k_lo + 1))
                hidden += bk - vis
    return hidden


# ------------------------------------------------------------------------- CPU baseline
def _stream_blocks(orc, q, kl, vl, mask, lay, blocks, causal):
    """psa_streaming's per-query-block loop (attention.py:171-218) over ``blocks``; returns the
    blocks' output rows and lse (the oracle restatement, one BLAS thread)."""
    import numpy as np
    scale = 1.0 / math.sqrt(lay.head_dim)
    outs, lses = [], []
    for i in blocks:
        qi = q[i * lay.q_block:(i + 1) * lay.q_block]
        m_run = np.full(lay.q_block, -np.inf)
        l_run = np.zeros(lay.q_block)
        acc = np.zeros((lay.q_block, lay.head_dim))
        for j in range(lay.n_k):
            h = int(mask[i, j])
            if h == 0:
                continue
            kb, vb = orc.pyramid_block(kl, lay, j, h), orc.pyramid_block(vl, lay, j, h)
            s_ = qi @ kb.T * scale + (h - 1) * orc.LN2
            if causal:
                vis = orc.causal_key_visibility(lay, i, j, h)
                if vis is not None:
                    s_ = np.where(vis, s_, -np.inf)
            m_new = np.maximum(s_.max(axis=1), m_run)
            dead = np.isneginf(m_new)
            shift = np.where(dead, 0.0, m_new)
            p_ = np.exp(s_ - shift[:, None])
            p_[np.isneginf(s_)] = 0.0
            alpha = np.where(dead, 0.0, np.exp(m_run - shift))
            l_run = l_run * alpha + p_.sum(axis=1)
            acc = acc * alpha[:, None] + p_ @ vb
            m_run = m_new
        alive = l_run > 0
        safe = np.where(alive, l_run, 1.0)
        outs.append(np.where(alive[:, None], acc / safe[:, None], 0.0))
        lses.append(np.where(alive, m_run + np.log(safe), -np.inf))
    return np.concatenate(outs), np.concatenate(lses)


def _cpu_worker(args):
    """The oracle port of the reference path (pyramid -> importance -> level map -> streaming
    attention) on one head, timed; with the GPU's results for the same head it also returns the
    parity numbers (level-map / plan mismatches, O and lse errors)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import numpy as np
    from oracle import psa_oracle as orc
    (q, k, v, lay_t, taus, blocks, causal, estimator, stride, sim, gpu) = args
    lay = orc.Layout(*lay_t)
    t0 = time.perf_counter()
    kl, vl = orc.build_pyramid(k, v, lay)
    if estimator == "antidiagonal":
        scores = orc.importance_antidiagonal(q, k, lay, stride)
    else:
        scores = orc.importance_sampled(q, k, lay, 8, 8, 0)
    m = orc.assign_threshold(scores, taus)
    if sim is not None:
        m = orc.combine_mask(m, orc.level_caps(k, lay, sim))
    if causal:
        m = orc.causal_premask(m, lay)
    t1 = time.perf_counter()
    out, lse = _stream_blocks(orc, q, kl, vl, m, lay, blocks, causal)
    t2 = time.perf_counter()
    counts = [int((m[blocks] == h).sum()) for h in range(lay.levels + 1)]
    par = None
    if gpu is not None:
        g_lm, g_out, g_lse = gpu
        rows = np.concatenate([np.arange(i * lay.q_block, (i + 1) * lay.q_block) for i in blocks])
        ref_o, ref_l = out, lse
        got_o, got_l = g_out[rows].astype(np.float64), g_lse[rows].astype(np.float64)
        fin = np.isfinite(ref_l)
        par = {"level_map_mismatches": int((g_lm != m).sum()), "level_map_entries": int(m.size),
               "o_rel_l2": float(np.linalg.norm(got_o - ref_o) / max(np.linalg.norm(ref_o), 1e-300)),
               "o_max_abs_over_max_ref": float(np.abs(got_o - ref_o).max() / max(np.abs(ref_o).max(), 1e-300)),
               "lse_max_abs": float(np.abs(got_l[fin] - ref_l[fin]).max()) if fin.any() else 0.0,
               "empty_rows_match": bool(np.array_equal(np.isfinite(got_l), fin))}
    return t1 - t0, t2 - t1, counts, par


def _head_worker(conn, data):
    """A persistent oracle worker: receives its head's inputs once, then a query-block list per
    step, and answers with _cpu_worker's result (so steps time the compute, not the transfer)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    conn.send("ready")
    while True:
        blocks = conn.recv()
        if blocks is None:
            break
        q, k, v, lay_t, taus, _, causal, est, stride, sim, gpu = data
        conn.send(_cpu_worker((q, k, v, lay_t, taus, blocks, causal, est, stride, sim, gpu)))
    conn.close()


class HeadWorkers:
    """One spawned process per head (one BLAS thread each) holding its data across steps."""

    def __init__(self, datas):
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        saved = {k_: os.environ.get(k_) for k_ in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS",
                                                    "MKL_NUM_THREADS")}
        for k_ in saved:  # children inherit: one BLAS thread per worker process
            os.environ[k_] = "1"
        try:
            self.conns, self.procs = [], []
            for d in datas:
                a, b = ctx.Pipe()
                p_ = ctx.Process(target=_head_worker, args=(b, d), daemon=True)
                p_.start()
                self.conns.append(a)
                self.procs.append(p_)
            for c in self.conns:  # started, data unpickled: the timed runs see compute only
                assert c.recv() == "ready"
        finally:
            for k_, v_ in saved.items():
                if v_ is None:
                    os.environ.pop(k_, None)
                else:
                    os.environ[k_] = v_

    def run(self, blocks):
        """Every worker streams ``blocks`` of its head; returns (results, wall seconds)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(list(blocks))
        res = [c.recv() for c in self.conns]
        return res, time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except (BrokenPipeError, EOFError, OSError):  # a worker that already died
                pass
        for p_ in self.procs:
            p_.join(timeout=30)
            if p_.is_alive():
                p_.terminate()


def cpu_baseline(cfg, q, k, v, gpu=None, blocks_per_head=None, max_workers=None):
    """The oracle port of the reference path on min(cores, heads) heads in parallel processes
    (one BLAS thread each). Each worker runs a WHOLE head (pyramid, importance, assignment and
    psa_streaming over every query block, or the first ``blocks_per_head`` blocks); the rate is the
    executed FLOPs of the heads run / wall time, and the per-forward time is extrapolated to all
    heads (BASELINE.md "CPU baseline"). ``gpu``: per worker head (level map, out, lse) of the GPU
    run, for the parity block. q/k/v: [1, heads, N, d] tensors holding heads 0..workers-1."""
    import numpy as np
    cores = os.cpu_count() or 1
    heads = q.shape[1]
    workers = max(1, min(cores, heads, max_workers or cores))
    N, bq = cfg["N"], cfg["b_q"]
    n_q = N // bq
    blocks = list(range(n_q if blocks_per_head is None else min(n_q, blocks_per_head)))
    lay_t = (N, cfg["d"], bq, cfg["b_k"], cfg["levels"])
    group = cfg["Hq"] // cfg["Hkv"]
    jobs = []
    for w in range(workers):
        hk = w // group
        jobs.append((q[0, w].to(torch_f64()).cpu().numpy(), k[0, hk].to(torch_f64()).cpu().numpy(),
                     v[0, hk].to(torch_f64()).cpu().numpy(), lay_t, cfg["taus"], blocks,
                     cfg["causal"], cfg["estimator"], cfg["stride"], cfg["sim"],
                     None if gpu is None else gpu[w]))
    hw = HeadWorkers(jobs)  # inputs (and the GPU results for the parity check) sent once
    res, wall = hw.run(blocks)
    hw.close()
    pre = statistics.mean(r[0] for r in res)
    att = statistics.mean(r[1] for r in res)
    flops = sum(flops_from_counts(r[2], cfg, 0) for r in res)
    if cfg["causal"]:
        flops -= 4 * cfg["d"] * workers * _causal_hidden_pairs_blocks(N, bq, cfg["b_k"], blocks)
    per_head = pre + att * (n_q / len(blocks))
    total_heads = cfg["B"] * cfg["Hq"]
    est_time = per_head * math.ceil(total_heads / workers)
    out = {
        "value": flops / wall / 1e12, "unit": "TFLOP/s", "cores": workers, "kind": "port",
        "cpu_model": cpu_model(), "host_cores": cores,
        "sample": (f"oracle (numpy fp64 restatement of pyrattn, one BLAS thread per process) on "
                   f"{workers} heads in parallel processes: per head pyramid + importance + level map "
                   f"({pre:.2f} s) + psa_streaming over {len(blocks)}/{n_q} query blocks "
                   f"({att:.2f} s); rate = executed FLOPs / wall ({wall:.1f} s); extrapolated "
                   f"{total_heads} heads = {est_time:.1f} s/forward"),
        "extrapolated_s_per_forward": est_time, "sample_wall_s": wall,
        "executed_tflop_sample": flops / 1e12,
    }
    if gpu is not None:
        pars = [r[3] for r in res]
        out["parity"] = {
            "heads": workers, "query_blocks_per_head": len(blocks),
            "level_map_mismatches": sum(p_["level_map_mismatches"] for p_ in pars),
            "level_map_entries": sum(p_["level_map_entries"] for p_ in pars),
            "o_rel_l2_max": max(p_["o_rel_l2"] for p_ in pars),
            "o_max_abs_over_max_ref": max(p_["o_max_abs_over_max_ref"] for p_ in pars),
            "lse_max_abs": max(p_["lse_max_abs"] for p_ in pars),
            "empty_rows_match": all(p_["empty_rows_match"] for p_ in pars),
            "vs": "oracle psa_streaming with the reference's fp64 pyramid (the GPU pools in fp64 and "
                  "stores bf16, so O/lse include the bf16 pyramid rounding; the tests bound the "
                  "kernel alone at rel-L2 <= 5e-3, lse <= 1e-3)"}
    return out


def torch_f64():
    import torch
    return torch.float64


# ------------------------------------------------------------------------- main
def self_launch(args):
    """--gpus N without a torchrun environment: re-exec under torch.distributed.run with N ranks
    on 127.0.0.1 (NCCL when the node has N GPUs; gloo with ranks sharing the GPUs otherwise)."""
    import socket
    import torch
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    if torch.cuda.device_count() < args.gpus:
        env.setdefault("PSA_BENCH_DIST_BACKEND", "gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-yardsticks", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    ngpu = max(1, torch.cuda.device_count())
    # NCCL needs one GPU per rank; with more ranks than GPUs (a functional multi-rank run on one
    # box) the ranks share GPUs over gloo and the line says so
    backend = os.environ.get("PSA_BENCH_DIST_BACKEND", "nccl" if ngpu >= world else "gloo")
    if not torch.cuda.is_available() and args.impl == "reference":  # the CPU arm runs anywhere
        device, backend = torch.device("cpu"), "gloo"
    else:
        device = torch.device(f"cuda:{local % ngpu}")
        torch.cuda.set_device(device)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    red_dev = device if backend == "nccl" else torch.device("cpu")

    if args.impl == "reference":
        return main_reference(args, cfg, rank, world, device)
    if args.config == "cfg5":
        return main_sweep(args, cfg, rank, world, device, red_dev)

    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200 import _lib
    from paper_2512_04025_b200.attention import attention_forward
    from paper_2512_04025_b200.importance import antidiagonal_scores, importance_scores
    from paper_2512_04025_b200.layout import LevelThresholds, SamplerConfig, SimThresholds
    from paper_2512_04025_b200.mask import assign_levels_device
    from paper_2512_04025_b200.parallel import gather_partitioned, partition, rank_cost
    from paper_2512_04025_b200.pyramid import build_pyramid, similarity_caps

    _lib.load()
    Hq, Hkv = cfg["Hq"], cfg["Hkv"]
    rc = run_config(cfg)
    lay = rc.layout()
    n_q = lay.n_q
    # (batch, head, query-block set) work units: heads cut into equal-cost query-block parts just
    # enough to divide evenly over the ranks (parallel.partition); no data-path collective
    calls = partition(Hq, Hkv, n_q, world, rank, cfg["causal"])
    segs = []
    for q_lo, q_hi, kv_lo, kv_hi, blocks in calls:
        qs, ks, vs = make_inputs(cfg, list(range(q_lo, q_hi)), list(range(kv_lo, kv_hi)), device)
        blk = None if blocks is None else torch.tensor(blocks, dtype=torch.int32, device=device)
        segs.append((qs, ks, vs, blk, blocks))
    sampler = SamplerConfig(8, 8, 0)
    rule = LevelThresholds(cfg["taus"])
    stream = torch.cuda.current_stream(device)
    sim = SimThresholds(cfg["sim"]) if cfg["sim"] else None
    stage_names = ("pyramid", "importance", "assign", "attention")
    # per call: pyramid 1; importance 6 (2 int8 slicers, xl_stats, xl_merge, the fp64 fallback
    # kernel that exits for unflagged heads, finalize); similarity caps 1 if on; assign 1;
    # attention 1
    launches_per_step = (1 + 6 + (1 if cfg["sim"] else 0) + 1 + 1) * len(segs)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        pyrs = [build_pyramid(ks, vs, lay) for _, ks, vs, _, _ in segs]
        capss = [similarity_caps(ks, lay, sim) if sim is not None else None for _, ks, _, _, _ in segs]
        if ev:
            ev[1].record(stream)
        if cfg["estimator"] == "antidiagonal":
            scores = [antidiagonal_scores(qs, ks, lay, cfg["stride"], qblocks=b_)
                      for qs, ks, _, b_, _ in segs]
        else:
            scores = [importance_scores(qs, ks, lay, sampler, "max", qblocks=b_)
                      for qs, ks, _, b_, _ in segs]
        if ev:
            ev[2].record(stream)
        plans = [assign_levels_device(sc, mode="threshold", rule=rule, levels=lay.levels,
                                      b_q=lay.q_block, b_k=lay.k_block, hkv=sg[1].shape[1],
                                      caps=cp, causal=cfg["causal"], qblocks=sg[3])
                 for sc, sg, cp in zip(scores, segs, capss)]
        if ev:
            ev[3].record(stream)
        outs = [attention_forward(sg[0], pyr, plan, cfg["causal"], qblocks=sg[3])
                for sg, pyr, plan in zip(segs, pyrs, plans)]
        if ev:
            ev[4].record(stream)
        return plans, outs

    for _ in range(max(args.warmup, 3)):
        plans, outs = step()
    torch.cuda.synchronize()
    # short configs: keep warming up (untimed) for >= 0.5 s so the SM clock has left its idle
    # state before the timed region
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.5:
        step()
        torch.cuda.synchronize()
    counts = sum(p_.level_counts for p_ in plans).cpu().tolist()
    flops_local = flops_from_counts(counts, cfg, 0)
    if cfg["causal"]:  # straddling level-1 pairs count only their visible (q, k) pairs
        for sg in segs:
            blk = range(n_q) if sg[4] is None else sg[4]
            flops_local -= 4 * cfg["d"] * cfg["B"] * sg[0].shape[1] * _causal_hidden_pairs_blocks(
                cfg["N"], cfg["b_q"], cfg["b_k"], blk)
    executed_tiles = sum(int(((p_.info[:, 1] + 127) // 128).sum()) for p_ in plans)
    if world > 1:  # whole-job level histogram
        ct = torch.tensor(counts + [executed_tiles], dtype=torch.int64, device=red_dev)
        dist.all_reduce(ct, op=dist.ReduceOp.SUM)
        counts, executed_tiles = ct[:-1].cpu().tolist(), int(ct[-1])
    rho_bar = psa.report_from_counts(counts, sum(counts)).rho_bar

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device.index) as clk:
        start.record(stream)
        for s_ in range(args.steps):
            plans, outs = step(evs[s_])
        end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_total = start.elapsed_time(end)
    stage_ms = {name: statistics.mean(evs[s_][i].elapsed_time(evs[s_][i + 1])
                                      for s_ in range(args.steps))
                for i, name in enumerate(stage_names)}
    stats = torch.tensor([ms_total, float(flops_local), stage_ms["attention"]], dtype=torch.float64,
                         device=red_dev)
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm_ = stats.clone()
        dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
        ms_total, flops_all, attn_ms_max = float(mx[0]), float(sm_[1]), float(mx[2])
    else:
        flops_all, attn_ms_max = float(flops_local), stage_ms["attention"]
    ms_step = ms_total / args.steps
    value = flops_all / (ms_step * 1e-3) / 1e12

    # ---- optional NCCL gather of O onto rank 0, timed separately
    gather = None
    if world > 1:
        pieces = [o[0] if backend == "nccl" else o[0].cpu() for o in outs]
        for _ in range(2):
            gather_partitioned(pieces, Hq, Hkv, n_q, lay.q_block, cfg["causal"], dst=0)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            full_o = gather_partitioned(pieces, Hq, Hkv, n_q, lay.q_block, cfg["causal"], dst=0)
        torch.cuda.synchronize()
        dist.barrier()
        g_ms = (time.perf_counter() - t0) * 1e3 / reps
        gt = torch.tensor([g_ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        out_bytes = cfg["B"] * Hq * cfg["N"] * cfg["d"] * 2
        gather = {"ms": round(float(gt[0]), 3), "bytes": out_bytes, "backend": backend,
                  "op": "dist.gather of every rank's O pieces onto rank 0 (padded flat buffers), "
                        "wall clock max over ranks, outside the timed region"}
        del full_o

    # ---- the same step replayed from a CUDA graph (graph.py: the chain is sync-free, so its host
    # work - argument checks, tensor maps, allocations, ctypes calls - is captured once)
    graph = None
    if world == 1:
        try:
            side = torch.cuda.Stream(device)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                step()
            stream.wait_stream(side)
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg):
                step()
            for _ in range(3):
                cg.replay()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            for _ in range(args.steps):
                cg.replay()
            b_.record(stream)
            torch.cuda.synchronize()
            g_ms = a_.elapsed_time(b_) / args.steps
            graph = {"ms_per_step": round(g_ms, 4),
                     "value": round(flops_all / (g_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                     "what": "the timed step's kernels captured once into a CUDA graph and "
                             "replayed (no per-call host work); same inputs and outputs; timed "
                             "right after the eager region, so on a hotter, possibly more "
                             "power-capped GPU (it matters for launch-bound shapes, not cfg3)"}
            del cg
        except Exception as exc:  # noqa: BLE001 - supplementary; must not kill the line
            graph = {"error": repr(exc)}

    # ---- end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(psa, rc, segs, args, stream, flops_all, world, device, red_dev)

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    achieved = float(flops_local) / (stage_ms["attention"] * 1e-3) / 1e12
    # tensor work the kernel executes incl. slot / row padding and the bias step: per 128-key
    # tile S (8 + 1 K-steps) and PV (8 K-steps) of 128 x 128 x 16 MMAs
    exec_flops = executed_tiles * 17 * 2 * 128 * 128 * 16
    traffic = None
    prof = ROOT / "profiles" / f"attention_ncu_summary_{args.config}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None

    yard = None
    if rank == 0 and world == 1 and not args.no_yardsticks and cfg["B"] == 1 and Hq == Hkv:
        yard = yardsticks(cfg, segs, lay, stream, attention_forward, psa)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import numpy as np
            qs, ks, vs = segs[0][0], segs[0][1], segs[0][2]
            workers = max(1, min(os.cpu_count() or 1, qs.shape[1]))
            lm = plans[0].level_map[0, :workers].cpu().numpy()
            o = outs[0][0][0, :workers].float().cpu().numpy()
            ls = outs[0][1][0, :workers].cpu().numpy()
            gpu = [(lm[h], o[h], ls[h]) for h in range(workers)]
            cpu = cpu_baseline(cfg, qs, ks, vs, gpu=gpu)
        except Exception as exc:  # noqa: BLE001 - the baseline must not kill the GPU line
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {exc!r}"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    costs = [rank_cost(partition(Hq, Hkv, n_q, world, r, cfg["causal"]), n_q, cfg["causal"])
             for r in range(world)]
    line = {
        "metric": "PSA fwd effective TFLOPS (and ms) at Wan2.1-14B 720p shape",
        "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic N(0,1) bf16 Q/K/V (seeded torch.Generator per head)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "B": cfg["B"], "Hq": Hq,
                   "Hkv": Hkv, "L": cfg["N"], "d": cfg["d"], "b_q": cfg["b_q"],
                   "b_k": cfg["b_k"], "levels": cfg["levels"],
                   "estimator": (f"antidiagonal stride {cfg['stride']} (fp64)"
                                 if cfg["estimator"] == "antidiagonal" else "sampled-max s_q=s_k=8 (fp64)"),
                   "sim_thresholds": cfg["sim"],
                   "mask": f"threshold taus={[round(t, 6) for t in cfg['taus']]}",
                   "rho_bar": rho_bar, "level_counts": counts, "causal": cfg["causal"],
                   "executed_tflop_per_step": flops_all / 1e12,
                   "parallelism": (f"(batch, head, query-block set) units over {world} rank(s): "
                                   f"{len(calls)} call(s) on rank 0, est. max/min rank cost "
                                   f"{max(costs) / min(costs):.3f}; no data-path collective"),
                   "dist_backend": backend if world > 1 else None,
                   "shared_gpus": world > ngpu,
                   "l2": "inputs (Q/K/V 2.3 GB at cfg3) exceed the 126 MB L2; no flush needed"},
        "stage_ms": {k_: round(v_, 4) for k_, v_ in stage_ms.items()},
        "roofline": {"bound": "tensor", "kernel": "psa_attn_pp2_kernel",
                     "achieved": round(achieved, 2), "peak": peak_burst, "unit": "TFLOP/s",
                     "frac": round(achieved / peak_burst, 4),
                     "peak_note": "MEASURED_PEAKS.json bf16_tflops (burst; the attention stage is a "
                                  "~25 ms kernel)",
                     "frac_of_sustained": round(achieved / peak_sus, 4), "traffic": traffic,
                     "executed_tflop_incl_padding_per_step": exec_flops / 1e12,
                     "executed_frac_of_burst": round(exec_flops / (attn_ms_max * 1e-3) / 1e12 / peak_burst, 4)
                     if world == 1 else None},
        "e2e": e2e,
        "graph": graph,
        "gather": gather,
        "yardsticks": yard,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "cpu_baseline": {k_: v_ for k_, v_ in cpu.items() if k_ != "parity"} if cpu else None,
        "parity": cpu.get("parity") if cpu else None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def yardsticks(cfg, segs, lay, stream, attention_forward, psa):
    """Dense yardsticks on the same heads: this kernel on an all-level-1 plan, and torch SDPA
    (backend recorded), each timed with CUDA events over 3 reps after a warm-up."""
    import torch
    from paper_2512_04025_b200.attention import _dense_layout
    from paper_2512_04025_b200.mask import plan_from_mask
    from paper_2512_04025_b200.pyramid import build_pyramid
    q, k, v = segs[0][0], segs[0][1], segs[0][2]
    B, H, N, d = q.shape
    dense_flops = 4.0 * N * N * d * B * H

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    dl = _dense_layout(N, d)
    pyr = build_pyramid(k, v, dl)
    plan = plan_from_mask(torch.ones(B, H, dl.n_q, dl.n_k, dtype=torch.int8, device=q.device), dl,
                          False, B, H)
    k_ms = timed(lambda: attention_forward(q, pyr, plan, False))
    del pyr, plan
    out = {"dense_tflop": dense_flops / 1e12,
           "psa_kernel_all_level1_ms": round(k_ms, 3),
           "psa_kernel_all_level1_tflops": round(dense_flops / (k_ms * 1e-3) / 1e12, 1)}
    from torch.nn.attention import SDPBackend, sdpa_kernel
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                s_ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
            out["torch_sdpa_backend"] = name
            out["torch_sdpa_ms"] = round(s_ms, 3)
            out["torch_sdpa_tflops"] = round(dense_flops / (s_ms * 1e-3) / 1e12, 1)
            break
        except Exception as exc:  # noqa: BLE001
            out[f"torch_sdpa_{name}_error"] = repr(exc)[:120]
    return out


def main_sweep(args, cfg, rank, world, device, red_dev):
    """cfg5: PSA forward at budgets b = 0.1..0.5 (quantile cutpoints (0.6b, b, 1.8b, 1.8b), the
    PSA-3 family: rho_bar = b), the binary block-sparse baseline at the same budgets (one level,
    cutpoint b), and dense attention (this kernel with every block at level 1, and torch SDPA as
    the external FlashAttention-style yardstick). Device time per full forward and per attention
    launch; heads sharded over ranks like the other configs."""
    import torch
    import torch.distributed as dist

    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200 import _lib
    from paper_2512_04025_b200.attention import attention_forward
    from paper_2512_04025_b200.parallel import shard_heads
    from paper_2512_04025_b200.pipeline import psa_forward_4d

    _lib.load()
    heads, kv_heads = shard_heads(cfg["Hq"], cfg["Hkv"], world, rank)
    has_work = bool(heads)
    if not has_work:
        heads, kv_heads = [0], [0]
    q, k, v = make_inputs(cfg, heads, kv_heads, device)
    stream = torch.cuda.current_stream(device)
    reps = max(1, args.steps)

    def timed(fn):
        for _ in range(max(args.warmup, 3)):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        a.record(stream)
        for _ in range(reps):
            if has_work:
                fn()
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def base_cfg(**kw):
        d = dict(n=cfg["N"], d=cfg["d"], b_q=cfg["b_q"], b_k=cfg["b_k"], levels=cfg["levels"],
                 estimator="sampled-max", s_q=8, s_k=8, seed=0, tile_len=128)
        d.update(kw)
        return psa.RunConfig.from_dict(d)

    rows = []
    clk = ClockSampler(device.index)
    clk.__enter__()
    for beta in (0.1, 0.2, 0.3, 0.4, 0.5):
        entry = {"budget": beta}
        for name, rc in (("psa", base_cfg(mask="quantile",
                                          cutpoints=[0.6 * beta, beta, 1.8 * beta, 1.8 * beta])),
                         ("binary", base_cfg(mask="quantile", cutpoints=[beta]))):
            res = psa_forward_4d(q, k, v, rc)
            counts = res.plan.level_counts.cpu().tolist()
            flops = flops_from_counts(counts, cfg, cfg["B"] * len(heads)) if has_work else 0
            ft = torch.tensor([float(flops)], dtype=torch.float64, device=red_dev)
            if world > 1:
                dist.all_reduce(ft, op=dist.ReduceOp.SUM)
            step_ms = timed(lambda rc=rc: psa_forward_4d(q, k, v, rc))
            attn_ms = timed(lambda res=res: attention_forward(q, res.pyramid, res.plan, False))
            entry[name] = {"ms_per_forward": round(step_ms, 4), "attention_ms": round(attn_ms, 4),
                           "rho_bar": psa.report_from_counts(counts, sum(counts)).rho_bar,
                           "executed_tflop": float(ft[0]) / 1e12,
                           "attention_tflops": round(float(ft[0]) / (attn_ms * 1e-3) / 1e12, 2)}
        rows.append(entry)
    dense_flops = 4.0 * cfg["N"] * cfg["N"] * cfg["d"] * cfg["B"] * cfg["Hq"]
    full_ms = timed(lambda: psa.full_attention(q, k, v))
    from torch.nn.attention import SDPBackend, sdpa_kernel
    sdpa_backend = "default"
    try:
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            sdpa_ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
        sdpa_backend = "cudnn"
    except Exception:  # noqa: BLE001
        sdpa_ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
    clk.__exit__(None, None, None)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    b02 = rows[1]["psa"]
    line = {
        "metric": "PSA fwd effective TFLOPS (and ms) at Wan2.1-14B 720p shape",
        "value": round(b02["executed_tflop"] / (b02["ms_per_forward"] * 1e-3), 3),
        "unit": "TFLOP/s", "n_gpus": world, "steps": reps, "warmup": max(args.warmup, 3),
        "ms_per_step": b02["ms_per_forward"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic N(0,1) bf16 Q/K/V (seeded torch.Generator per head)",
        "config": {"workload": f"cfg5: {cfg['desc']}", "L": cfg["N"], "Hq": cfg["Hq"],
                   "d": cfg["d"], "b": cfg["b_q"], "value_at_budget": 0.2,
                   "parallelism": f"heads sharded over {world} GPU(s)"},
        "sweep": rows,
        "dense": {"tflop": dense_flops / 1e12,
                  "psa_kernel_all_level1_ms": round(full_ms, 4),
                  "psa_kernel_all_level1_tflops": round(dense_flops / (full_ms * 1e-3) / 1e12, 2),
                  "torch_sdpa_ms": round(sdpa_ms, 4), "torch_sdpa_backend": sdpa_backend,
                  "torch_sdpa_tflops": round(dense_flops / (sdpa_ms * 1e-3) / 1e12, 2)},
        "clocks": clk.summary(),
        "gpu_launches": None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(psa, rc, segs, args, stream, flops_all, world, device, red_dev=None):
    """Same metric through the public call a user makes with host data: psa.psa_attention on
    pinned host Q/K/V returns O and lse in pinned host memory (one call per work unit of the rank,
    with its query-block list). Every timed step includes the H2D of Q/K/V and the D2H of O/lse
    (the call pipelines head groups over copy-in / compute / copy-out streams, staging.py)."""
    import torch
    import torch.distributed as dist
    host = [tuple(x.cpu().pin_memory() for x in sg[:3]) for sg in segs]
    lay = rc.layout()
    outs = []
    for (hq, _, _), sg in zip(host, segs):
        rows = hq.shape[2] if sg[4] is None else len(sg[4]) * lay.q_block
        outs.append((torch.empty(hq.shape[:2] + (rows, hq.shape[3]), dtype=torch.bfloat16).pin_memory(),
                     torch.empty(hq.shape[:2] + (rows,), dtype=torch.float32).pin_memory()))

    per_group = int(os.environ["PSA_E2E_GROUP"]) if os.environ.get("PSA_E2E_GROUP") else None

    def one():
        for (hq, hk, hv), (out_h, lse_h), sg in zip(host, outs, segs):
            psa.psa_attention(hq, hk, hv, rc, device=device, out=out_h, lse=lse_h,
                              kv_heads_per_group=per_group, qblocks=sg[4])

    t_w = time.perf_counter()
    for w in range(1000):  # >= 2 untimed calls and >= 0.5 s (clocks out of their idle state)
        one()
        torch.cuda.synchronize()
        if w >= 1 and time.perf_counter() - t_w >= 0.5:
            break
    steps = max(1, args.steps)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    a.record(stream)
    for _ in range(steps):
        one()
    b.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / steps
    ms = a.elapsed_time(b) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev or device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    # PCIe floor of the same step: the H2D of Q/K/V alone (pinned, one stream)
    srcs = [x for sg in host for x in sg]
    dq = [torch.empty_like(x, device=device) for x in srcs]
    a.record(stream)
    for _ in range(steps):
        for dst, src in zip(dq, srcs):
            dst.copy_(src, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    h2d_ms = a.elapsed_time(b) / steps
    del dq
    return {"value": round(flops_all / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
            "h2d_only_ms": round(h2d_ms, 3),
            "ms_per_step": round(ms, 3), "host_wall_ms_per_step": round(wall, 3), "steps": steps,
            "api": "psa_attention(pinned host q, k, v[, qblocks]) -> host out, lse (staged "
                   "H2D/compute/D2H)",
            "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in srcs)),
            "d2h_bytes_per_step": int(sum(o.numel() * o.element_size() + l_.numel() * l_.element_size()
                                          for o, l_ in outs))}


def main_reference(args, cfg, rank, world, device):
    """--impl reference: the reference path's CPU implementation (the oracle port, numpy fp64, one
    BLAS thread per process) on every host core, same config/metric/unit; rank 0 only. Nothing
    from the GPU package runs here: inputs are synthesised with torch's RNG (the same per-head
    streams as our arm) and the executed FLOPs come from the oracle's own level maps.
    Each step is a bounded, fully timed sample: every worker runs one head's pyramid, importance
    and level map and streams the next ``nb`` query blocks of that head. The rate charges the
    per-head pre-work pro rata (nb / n_q of it, as a whole-head run amortises it); ms_per_step is
    the measured wall time of a step."""
    import torch
    import torch.distributed as dist
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    workers = min(cores, cfg["B"] * cfg["Hq"])
    heads = list(range(workers))
    group = cfg["Hq"] // cfg["Hkv"]
    kvh = sorted({h // group for h in heads})
    gen_dev = device if torch.cuda.is_available() else torch.device("cpu")
    q, k, v = make_inputs(cfg, heads, kvh, gen_dev)
    N, bq = cfg["N"], cfg["b_q"]
    n_q = N // bq
    nb = max(1, min(n_q, int(3.0e6 / N)))
    lay_t = (N, cfg["d"], bq, cfg["b_k"], cfg["levels"])
    data = [(q[0, h].double().cpu().numpy(), k[0, kvh.index(h // group)].double().cpu().numpy(),
             v[0, kvh.index(h // group)].double().cpu().numpy()) for h in heads]
    walls, rates, last = [], [], None
    hw = HeadWorkers([d_ + (lay_t, cfg["taus"], None, cfg["causal"], cfg["estimator"], cfg["stride"],
                            cfg["sim"], None) for d_ in data])  # head data sent once, untimed
    try:
        for s_ in range(max(args.warmup, 0) + args.steps):
            blocks = [(s_ * nb + b_) % n_q for b_ in range(nb)]
            res, wall = hw.run(blocks)
            pre = statistics.mean(r_[0] for r_ in res)
            flops = sum(flops_from_counts(r_[2], cfg, 0) for r_ in res)
            if cfg["causal"]:
                flops -= 4 * cfg["d"] * workers * _causal_hidden_pairs_blocks(N, bq, cfg["b_k"], blocks)
            charged = wall - pre * (1.0 - nb / n_q)
            if s_ >= args.warmup:
                walls.append(wall)
                rates.append(flops / charged / 1e12)
            last = (pre, wall, flops)
    finally:
        hw.close()
    value = statistics.mean(rates)
    ms_step = statistics.mean(walls) * 1e3
    sample = (f"oracle port (numpy fp64 restatement of pyrattn) on {workers} processes x 1 BLAS "
              f"thread ({cpu_model()}): per step every process runs one head's pyramid + "
              f"importance + level map ({last[0]:.2f} s) and psa_streaming over {nb}/{n_q} query "
              f"blocks; rate = executed FLOPs / (wall - pre-work * (1 - {nb}/{n_q}))")
    line = {
        "impl": "reference", "metric": "PSA fwd effective TFLOPS (and ms) at Wan2.1-14B 720p shape",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1) bf16-rounded Q/K/V",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "B": cfg["B"], "Hq": cfg["Hq"],
                   "Hkv": cfg["Hkv"], "L": cfg["N"], "d": cfg["d"], "b_q": cfg["b_q"],
                   "b_k": cfg["b_k"], "levels": cfg["levels"], "causal": cfg["causal"],
                   "executed_tflop_per_step": last[2] / 1e12,
                   "step": f"{workers} heads x {nb} query blocks (a bounded sample of the workload)"},
        "cpu_baseline": {"kind": "port", "cores": workers, "host_cores": cores,
                         "cpu_model": cpu_model(), "sample": sample, "value": value,
                         "unit": "TFLOP/s"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

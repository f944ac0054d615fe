"""Shared test helpers: seeded bf16 inputs seen identically by the GPU and the oracle."""

import numpy as np
import torch


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round to bf16 (RNE) and return as float64 — exactly what the GPU receives."""
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16) \
        .to(torch.float64).numpy()


def gaussian_qkv(seed: int, heads: int, n: int, d: int, kv_heads: int | None = None):
    """Q [heads, n, d], K/V [kv_heads, n, d] bf16-rounded float64 arrays."""
    kv_heads = heads if kv_heads is None else kv_heads
    rng = np.random.default_rng(seed)
    q = bf16_round(rng.standard_normal((heads, n, d), dtype=np.float32))
    k = bf16_round(rng.standard_normal((kv_heads, n, d), dtype=np.float32))
    v = bf16_round(rng.standard_normal((kv_heads, n, d), dtype=np.float32))
    return q, k, v


def correlated_qkv(seed: int, heads: int, g0: int, g1: int, d: int):
    """Smooth 2D random-walk fields (the reference's 'correlated' generator, pipeline.py:153-164)
    rounded to bf16: high adjacent-key similarity, large logits."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(3):
        per = []
        for _h in range(heads):
            mu = rng.normal(size=d) * 2.0
            w0 = np.cumsum(rng.normal(size=(g0, d)) * 0.25, axis=0)
            w1 = np.cumsum(rng.normal(size=(g1, d)) * 0.25, axis=0)
            per.append((mu[None, None] + w0[:, None] + w1[None, :]).reshape(g0 * g1, d))
        out.append(bf16_round(np.stack(per)))
    return out


def to_dev(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    den = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / den if den > 0 else float(np.linalg.norm(a))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns of float64 values (RNE)."""
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).view(torch.int16).numpy()


GOLDEN_DIR = __import__("pathlib").Path(__file__).resolve().parent / "golden"
GOLDEN_CASES = sorted(p.stem for p in GOLDEN_DIR.glob("*.npz") if p.stem not in ("hilbert_orders", "schedules", "pipeline_report", "psat_files"))


def load_golden(name: str) -> dict:
    """Golden case produced by the reference (tests/golden/make_golden.py)."""
    z = np.load(GOLDEN_DIR / f"{name}.npz", allow_pickle=False)
    g = {key: z[key] for key in z.files}
    for key in ("q", "k", "v"):
        g[key] = torch.from_numpy(g[key].view(np.int16)).view(torch.bfloat16) \
            .to(torch.float64).numpy()
    g["cfg"] = eval(str(g["config"]))  # repr of a plain dict written by make_golden.py
    g["lay"] = tuple(int(x) for x in g["layout"])
    return g

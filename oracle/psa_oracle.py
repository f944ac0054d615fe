"""CPU ORACLE — test infrastructure only, never the product path.

A plain numpy/float64 restatement of the reference PSA forward path (`pyrattn` 0.1.0 at
/root/reference/pkg/src/pyrattn). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module, and only as the checker (or the
timed CPU baseline). Each function cites the reference file:line it restates.

Pinning: tests/test_oracle_golden.py checks every function here against golden vectors
produced by the reference itself (tests/golden/make_golden.py imports pyrattn from
/root/reference in the build container) and against the reference's own known-answer tests
(listed in SURVEY.md §4). Numerics follow the reference exactly: fp64 everywhere, the same
numpy calls in the same order where the result depends on rounding (softmax, fsum,
Neumaier, pairwise means).
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

LN2 = math.log(2.0)


# --------------------------------------------------------------------------- layout
class Layout:
    """blocks.py:13-64 — divisibility rules of BlockLayout."""

    def __init__(self, seq_len, head_dim, q_block, k_block, levels):
        if min(seq_len, head_dim, q_block, k_block) < 1 or levels < 1:
            raise ValueError("layout dimensions must be positive")
        if seq_len % q_block or seq_len % k_block:
            raise ValueError("seq_len not divisible by the block sizes")
        if k_block % (1 << (levels - 1)):
            raise ValueError("k_block not divisible by 2^(levels-1)")
        self.seq_len, self.head_dim = seq_len, head_dim
        self.q_block, self.k_block, self.levels = q_block, k_block, levels
        self.n_q, self.n_k = seq_len // q_block, seq_len // k_block

    def pooled_len(self, h):
        return self.k_block >> (h - 1)


# --------------------------------------------------------------------------- pyramid
def mean_pool_rows(x):
    """linalg.py:46-58 — 0.5*(x[2t] + x[2t+1]); an odd last row passes through."""
    n = x.shape[0]
    half = n // 2
    out = 0.5 * (x[0:2 * half:2] + x[1:2 * half:2])
    return np.vstack([out, x[-1:]]) if n % 2 else out


def build_pyramid(k, v, lay):
    """blocks.py:86-109. Returns per-level arrays (n_k * L_h, d) for K and V; level 1 = raw.

    Blocks start at multiples of b_k and b_k is a multiple of 2^(H-1), so pooling the whole
    sequence pairwise is the same op sequence as pooling each block separately.
    """
    ks, vs = [np.asarray(k, np.float64)], [np.asarray(v, np.float64)]
    for _ in range(lay.levels - 1):
        ks.append(mean_pool_rows(ks[-1]))
        vs.append(mean_pool_rows(vs[-1]))
    return ks, vs


def pyramid_block(levels_arr, lay, j, h):
    L = lay.pooled_len(h)
    return levels_arr[h - 1][j * L:(j + 1) * L]


# --------------------------------------------------------------------------- importance
def row_softmax(a):
    """linalg.py:38-43."""
    shifted = a - a.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=1, keepdims=True)


def sample_rows(lay, s_q, s_k, seed):
    """importance.py:68-76 — one generator: every query block, then every KV block."""
    rng = np.random.default_rng(seed)
    q_rows = [i * lay.q_block + rng.permutation(lay.q_block)[:s_q] for i in range(lay.n_q)]
    k_rows = [j * lay.k_block + rng.permutation(lay.k_block)[:s_k] for j in range(lay.n_k)]
    return np.concatenate(q_rows), np.concatenate(k_rows)


def importance_sampled(q, k, lay, s_q, s_k, seed, reducer="max"):
    """importance.py:52-85."""
    qr, kr = sample_rows(lay, s_q, s_k, seed)
    probs = row_softmax(q[qr] @ k[kr].T / math.sqrt(lay.head_dim))
    blocks = probs.reshape(lay.n_q, s_q, lay.n_k, s_k)
    return blocks.max(axis=(1, 3)) if reducer == "max" else blocks.mean(axis=(1, 3))


def importance_antidiagonal(q, k, lay, stride):
    """importance.py:97-132 — per query block the full b_q x N logits (multiply by 1/sqrt(d)),
    the (p + c) % stride == 0 picks, a row softmax across all blocks, mass per block, mean."""
    per = lay.k_block // stride
    scale = 1.0 / math.sqrt(lay.head_dim)
    cols = np.stack([np.arange((-p) % stride, lay.k_block, stride) for p in range(lay.q_block)])
    all_cols = (cols[:, None, :] + np.arange(lay.n_k)[None, :, None] * lay.k_block
                ).reshape(lay.q_block, -1)
    out = np.empty((lay.n_q, lay.n_k))
    for i in range(lay.n_q):
        logits = q[i * lay.q_block:(i + 1) * lay.q_block] @ k.T * scale
        picked = np.take_along_axis(logits, all_cols, axis=1)
        out[i] = row_softmax(picked).reshape(lay.q_block, lay.n_k, per).sum(axis=2).mean(axis=0)
    return out


# --------------------------------------------------------------------------- mask
def descending_order(s):
    """mask.py:107-109 — stable argsort of -s."""
    return np.argsort(-s, axis=1, kind="stable")


def neumaier_cumsum(vec):
    """mask.py:112-125 — sequential Neumaier running sums, out[i] = total + comp."""
    out = np.empty_like(vec)
    total = comp = 0.0
    for i, x in enumerate(vec):
        t = total + x
        comp += ((total - t) + x) if abs(total) >= abs(x) else ((x - t) + total)
        total = t
        out[i] = total + comp
    return out


def assign_threshold(scores, taus):
    """mask.py:128-151 (Alg. 2)."""
    s = np.asarray(scores, np.float64)
    taus = np.asarray(taus, np.float64)
    n_q, n_k = s.shape
    order = descending_order(s)
    lev = np.empty((n_q, n_k), dtype=np.int64)
    for i in range(n_q):
        row = s[i, order[i]]
        tot = math.fsum(row)
        e = row / tot if tot > 0 else np.full(n_k, 1.0 / n_k)
        cum = np.minimum(neumaier_cumsum(e), 1.0)
        idx = np.searchsorted(taus, cum, side="left")
        lev[i, order[i]] = np.where(idx < len(taus), idx + 1, 0)
    return lev


def binary_mask(scores, tau):
    """mask.py:154-158."""
    return assign_threshold(scores, (tau,))


def fraction_counts(points, n_k):
    """mask.py:161-164."""
    c = [min(n_k, int(math.floor(p * n_k + 0.5))) for p in points]
    return np.maximum.accumulate(np.asarray(c, dtype=np.int64))


def assign_quantile(scores, points):
    """mask.py:167-179."""
    s = np.asarray(scores, np.float64)
    n_q, n_k = s.shape
    counts = fraction_counts(points, n_k)
    order = descending_order(s)
    idx = np.searchsorted(counts, np.arange(n_k), side="right")
    lev_sorted = np.where(idx < len(counts), idx + 1, 0)
    lev = np.empty((n_q, n_k), dtype=np.int64)
    np.put_along_axis(lev, order, np.broadcast_to(lev_sorted, (n_q, n_k)), axis=1)
    return lev


PRESETS = {
    "psa-1": (0.25, 0.25, 0.25, 0.25), "psa-2": (0.0, 0.0, 1.0, 1.0),
    "psa-3": (0.15, 0.25, 0.45, 0.45), "psa-4": (0.10, 0.30, 0.50, 0.50),
    "psa-5": (0.10, 0.20, 0.60, 0.60),
}


def strided_block_similarity(block, stride):
    """mask.py:182-195 — mean clipped cosine of row pairs `stride` apart; None if none."""
    if block.shape[0] <= stride:
        return None
    a, b = block[:-stride], block[stride:]
    na, nb = np.linalg.norm(a, axis=1), np.linalg.norm(b, axis=1)
    ok = (na > 0) & (nb > 0)
    if not ok.any():
        return None
    cos = (a[ok] * b[ok]).sum(axis=1) / (na[ok] * nb[ok])
    return float(np.clip(cos, -1.0, 1.0).mean())


def level_caps(k, lay, sim_taus):
    """mask.py:198-234 — caps start at 1, max over levels whose similarity > tau (strict)."""
    caps = np.ones(lay.n_k, dtype=np.int64)
    for j in range(lay.n_k):
        blk = k[j * lay.k_block:(j + 1) * lay.k_block]
        for h in range(2, lay.levels + 1):
            sim = strided_block_similarity(blk, 1 << (h - 1))
            if sim is not None and sim > sim_taus[h - 2]:
                caps[j] = max(caps[j], h)
    return caps


def combine_mask(mask, caps):
    """mask.py:237-247."""
    return np.minimum(np.asarray(mask, np.int64), np.asarray(caps, np.int64)[None, :])


def causal_premask(mask, lay):
    """mask.py:324-349."""
    m = np.asarray(mask, np.int64).copy()
    i = np.arange(lay.n_q)[:, None]
    j = np.arange(lay.n_k)[None, :]
    future = j * lay.k_block > (i + 1) * lay.q_block - 1
    visible = (j + 1) * lay.k_block - 1 <= i * lay.q_block
    m[future] = 0
    m[~future & ~visible] = 1
    return m


def report_from_counts(counts, total):
    """mask.py:278-300 — exact rationals rounded once."""
    counts = [int(c) for c in counts]
    rho = sum((Fraction(counts[h], total) * Fraction(1, 1 << (h - 1))
               for h in range(1, len(counts))), Fraction(0))
    return {"level_counts": counts, "total_entries": total, "rho_bar": float(rho),
            "sparsity": float(1 - rho), "kv_coverage": float(Fraction(total - counts[0], total)),
            "level_histogram": [float(Fraction(c, total)) for c in counts]}


def sparsity_report(mask, levels):
    """mask.py:303-321."""
    m = np.asarray(mask, np.int64)
    return report_from_counts([int((m == h).sum()) for h in range(levels + 1)], m.size)


# --------------------------------------------------------------------------- attention
def causal_key_visibility(lay, i, j, h):
    """attention.py:88-108 — None if fully visible, else (b_q, rows) k_pos <= q_pos mask."""
    q_lo, q_hi = i * lay.q_block, (i + 1) * lay.q_block - 1
    k_lo, k_hi = j * lay.k_block, (j + 1) * lay.k_block - 1
    if k_hi <= q_lo:
        return None
    if h != 1:
        raise ValueError(f"causal mode requires level 1 on straddling pair ({i}, {j})")
    return np.arange(k_lo, k_hi + 1)[None, :] <= np.arange(q_lo, q_hi + 1)[:, None]


def psa_streaming(q, kl, vl, mask, lay, causal=False):
    """attention.py:171-218 — block-by-block online softmax in ascending j.

    Returns (out (N, d), lse (N,), skipped_rows)."""
    q = np.asarray(q, np.float64)
    m = np.asarray(mask, np.int64)
    scale = 1.0 / math.sqrt(lay.head_dim)
    out = np.zeros((lay.seq_len, lay.head_dim))
    lse = np.full(lay.seq_len, -np.inf)
    skipped = 0
    for i in range(lay.n_q):
        rows = slice(i * lay.q_block, (i + 1) * lay.q_block)
        qi = q[rows]
        m_run = np.full(lay.q_block, -np.inf)
        l_run = np.zeros(lay.q_block)
        acc = np.zeros((lay.q_block, lay.head_dim))
        for j in range(lay.n_k):
            h = int(m[i, j])
            if h == 0:
                continue
            kb, vb = pyramid_block(kl, lay, j, h), pyramid_block(vl, lay, j, h)
            s = qi @ kb.T * scale + (h - 1) * LN2
            if causal:
                vis = causal_key_visibility(lay, i, j, h)
                if vis is not None:
                    s = np.where(vis, s, -np.inf)
            m_new = np.maximum(s.max(axis=1), m_run)
            dead = np.isneginf(m_new)
            shift = np.where(dead, 0.0, m_new)
            p = np.exp(s - shift[:, None])
            p[np.isneginf(s)] = 0.0
            alpha = np.where(dead, 0.0, np.exp(m_run - shift))
            l_run = l_run * alpha + p.sum(axis=1)
            acc = acc * alpha[:, None] + p @ vb
            m_run = m_new
        alive = l_run > 0
        skipped += int((~alive).sum())
        safe = np.where(alive, l_run, 1.0)
        out[rows] = np.where(alive[:, None], acc / safe[:, None], 0.0)
        lse[rows] = np.where(alive, m_run + np.log(safe), -np.inf)
    return out, lse, skipped


def psa_materialized(q, kl, vl, mask, lay, causal=False, rows_of=None):
    """attention.py:120-168 (psa_reference) — per query block, concatenate the selected pooled
    segments and softmax once. Equal to psa_streaming to ~1e-12; used for large parity checks.
    ``rows_of`` optionally restricts the query blocks evaluated (others stay zero / nan)."""
    q = np.asarray(q, np.float64)
    m = np.asarray(mask, np.int64)
    scale = 1.0 / math.sqrt(lay.head_dim)
    out = np.zeros((lay.seq_len, lay.head_dim))
    lse = np.full(lay.seq_len, -np.inf)
    skipped = 0
    blocks = range(lay.n_q) if rows_of is None else rows_of
    for i in blocks:
        rows = slice(i * lay.q_block, (i + 1) * lay.q_block)
        sel = np.nonzero(m[i])[0]
        if sel.size == 0:
            skipped += lay.q_block
            continue
        ks, vs, bias, vis_parts = [], [], [], []
        for j in sel:
            h = int(m[i, j])
            kb = pyramid_block(kl, lay, j, h)
            ks.append(kb)
            vs.append(pyramid_block(vl, lay, j, h))
            bias.append(np.full(kb.shape[0], (h - 1) * LN2))
            if causal:
                vis = causal_key_visibility(lay, i, j, h)
                vis_parts.append(np.ones((lay.q_block, kb.shape[0]), bool) if vis is None else vis)
        s = q[rows] @ np.concatenate(ks).T * scale + np.concatenate(bias)[None, :]
        if causal:
            s = np.where(np.concatenate(vis_parts, axis=1), s, -np.inf)
        mx = s.max(axis=1)
        alive = np.isfinite(mx)
        skipped += int((~alive).sum())
        shift = np.where(alive, mx, 0.0)
        p = np.exp(s - shift[:, None])
        p[~np.isfinite(s)] = 0.0
        den = p.sum(axis=1)
        safe = np.where(alive, den, 1.0)
        out[rows] = np.where(alive[:, None], (p @ np.concatenate(vs)) / safe[:, None], 0.0)
        lse[rows] = np.where(alive, shift + np.log(safe), -np.inf)
    return out, lse, skipped


def full_attention(q, k, v):
    """attention.py:47-63."""
    s = q @ k.T / math.sqrt(q.shape[1])
    mx = s.max(axis=1)
    lse = mx + np.log(np.exp(s - mx[:, None]).sum(axis=1))
    return row_softmax(s) @ v, lse


def causal_full_attention(q, k, v):
    """attention.py:221-241."""
    n = q.shape[0]
    s = q @ k.T / math.sqrt(q.shape[1])
    s = np.where(np.tril(np.ones((n, n), dtype=bool)), s, -np.inf)
    mx = s.max(axis=1)
    p = np.exp(s - mx[:, None])
    p[np.isneginf(s)] = 0.0
    den = p.sum(axis=1)
    return (p @ v) / den[:, None], mx + np.log(den)


# --------------------------------------------------------------------------- permutation
def _sgn(v):
    return (v > 0) - (v < 0)


def _gilbert(x, y, ax, ay, bx, by):
    """permute.py:46-90 — generalized Hilbert walk, recursive as in the reference."""
    w, h = abs(ax + ay), abs(bx + by)
    dax, day, dbx, dby = _sgn(ax), _sgn(ay), _sgn(bx), _sgn(by)
    if h == 1:
        return [(x + t * dax, y + t * day) for t in range(w)]
    if w == 1:
        return [(x + t * dbx, y + t * dby) for t in range(h)]
    ax2, ay2, bx2, by2 = ax // 2, ay // 2, bx // 2, by // 2
    w2, h2 = abs(ax2 + ay2), abs(bx2 + by2)
    if 2 * w > 3 * h:
        if (w2 % 2) and w > 2:
            ax2, ay2 = ax2 + dax, ay2 + day
        return (_gilbert(x, y, ax2, ay2, bx, by)
                + _gilbert(x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by))
    if (h2 % 2) and h > 2:
        bx2, by2 = bx2 + dbx, by2 + dby
    return (_gilbert(x, y, bx2, by2, ax2, ay2)
            + _gilbert(x + bx2, y + by2, ax, ay, bx - bx2, by - by2)
            + _gilbert(x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby),
                       -bx2, -by2, -(ax - ax2), -(ay - ay2)))


def hilbert_order(grid):
    """permute.py:97-128 — flat token order along the 2D curve / 3D serpentine of 2D curves."""
    def walk(n0, n1):
        if n0 >= n1:
            return _gilbert(0, 0, n0, 0, 0, n1)
        return [(x, y) for (y, x) in _gilbert(0, 0, n1, 0, 0, n0)]
    grid = [int(g) for g in grid]
    if len(grid) == 2:
        return np.array([x * grid[1] + y for (x, y) in walk(*grid)], dtype=np.int64)
    n0, n1, n2 = grid
    plane, flat = walk(n1, n2), []
    for s in range(n0):
        if s:
            plane = plane[::-1]
        flat.extend(s * n1 * n2 + x * n2 + y for (x, y) in plane)
    return np.array(flat, dtype=np.int64)


# --------------------------------------------------------------------------- composition
def run_head(q, k, v, lay, *, estimator="sampled-max", s_q=None, s_k=None, seed=None,
             stride=None, mask="threshold", thresholds=None, cutpoints=None, tau=None,
             sim_thresholds=None, causal=False, executor="streaming", rows_of=None,
             grid=None, unpermute=False):
    """pipeline.py:256-314 stage order (with the optional curve permutation) without the
    scheduler and dense oracle. With ``unpermute`` both out and lse return in input order.

    Returns dict(scores, mask, caps, out, lse, skipped, report)."""
    q, k, v = (np.asarray(x, np.float64) for x in (q, k, v))
    perm = None
    if grid is not None:
        perm = hilbert_order(grid)
        q, k, v = q[perm], k[perm], v[perm]
    kl, vl = build_pyramid(k, v, lay)
    if estimator == "antidiagonal":
        scores = importance_antidiagonal(q, k, lay, stride)
    else:
        scores = importance_sampled(q, k, lay, s_q, s_k, seed,
                                    "max" if estimator == "sampled-max" else "mean")
    if mask == "threshold":
        m = assign_threshold(scores, thresholds)
    elif mask == "binary":
        m = binary_mask(scores, tau)
    else:
        m = assign_quantile(scores, cutpoints if mask == "quantile" else PRESETS[mask])
    caps = None
    if sim_thresholds is not None:
        caps = level_caps(k, lay, sim_thresholds)
        m = combine_mask(m, caps)
    if causal:
        m = causal_premask(m, lay)
    if executor == "streaming":
        out, lse, skipped = psa_streaming(q, kl, vl, m, lay, causal)
    else:
        out, lse, skipped = psa_materialized(q, kl, vl, m, lay, causal, rows_of=rows_of)
    if perm is not None and unpermute:
        inv = np.empty_like(perm)
        inv[perm] = np.arange(perm.size)
        out, lse = out[inv], lse[inv]
    return {"scores": scores, "mask": m, "caps": caps, "out": out, "lse": lse,
            "skipped": skipped, "report": sparsity_report(m, lay.levels), "pyramid": (kl, vl)}


def executed_flops(mask, lay, causal=False):
    """Algorithmic FLOPs of the executor: 4*d*sum over selected (i, j) of b_q * L_h
    (non-causal); causal counts only visible (query, key) pairs of straddling blocks."""
    m = np.asarray(mask, np.int64)
    total = 0
    for h in range(1, lay.levels + 1):
        cnt = int((m == h).sum())
        total += cnt * lay.q_block * lay.pooled_len(h)
    if causal:
        # subtract invisible pairs of straddling level-1 blocks
        for i in range(lay.n_q):
            for j in range(lay.n_k):
                if m[i, j] == 1:
                    vis = causal_key_visibility(lay, i, j, 1)
                    if vis is not None:
                        total -= int((~vis).sum())
    return 4 * lay.head_dim * total

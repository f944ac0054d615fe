"""How many level-map rows would a relative score error eps make uncertain (CPU, oracle)?
For each row: sorted scores s (desc), cum = cumsum / total. Block at sorted position k has true
cumulative sum within [(cum_{a-1} + s_k/T)(1-3eps), cum_b (1+3eps)] where [a, b] is the run of
positions whose scores lie within a factor (1 +- 4eps) of s_k; the row is fragile if some tau lies
inside some block's interval."""
import sys, time, math
import numpy as np
sys.path.insert(0, '/root/repo')
from oracle import psa_oracle as orc


def fragile_rows(scores, taus, eps):
    out = np.zeros(scores.shape[0], bool)
    taus = np.asarray(taus)
    for i, row in enumerate(scores):
        s = np.sort(row)[::-1]
        tot = s.sum()
        if tot <= 0:
            continue
        cum = np.cumsum(s) / tot
        prev = np.concatenate([[0.0], cum[:-1]])
        # window [a, b]: scores within relative 4 eps of s_k (s descending)
        a = np.searchsorted(-s, -s * (1 + 4 * eps), side='left')
        b = np.searchsorted(-s, -s * (1 - 4 * eps), side='right') - 1
        lo = (prev[a] + s / tot) * (1 - 3 * eps)
        hi = cum[b] * (1 + 3 * eps)
        for t in taus:
            if np.any((lo <= t) & (t <= hi)):
                out[i] = True
                break
    return out


def gauss(rng, n, d):
    x = rng.standard_normal((n, d)).astype(np.float32)
    u = x.view(np.uint32)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(1)
    alpha = 0.4673
    wan = (alpha * 0.35, alpha * 0.6, alpha * 0.8, 0.95)
    a4 = 0.431938
    cfg4 = tuple(a4 * t for t in (0.35, 0.6, 0.8, 0.95))
    cases = [("cfg3 sampled", 75600, 120, wan, None), ("cfg4 antidiag", 32768, 128, cfg4, 8)]
    which = sys.argv[1:] or ["cfg3", "cfg4"]
    for name, n, bq, taus, stride in cases:
        if name.split()[0] not in which:
            continue
        lay = orc.Layout(n, 128, bq, 120 if stride is None else 64, 4)
        q, k = gauss(rng, n, 128), gauss(rng, n, 128)
        t0 = time.time()
        s = (orc.importance_sampled(q, k, lay, 8, 8, 0) if stride is None
             else orc.importance_antidiagonal(q, k, lay, stride))
        t1 = time.time()
        for eps in (3e-6, 1e-5, 3e-5, 1e-4):
            f = fragile_rows(s, taus, eps)
            print(f"{name}: n_q={s.shape[0]} n_k={s.shape[1]} eps={eps:g}: fragile rows "
                  f"{f.sum()} ({f.mean():.2%})  [scores {t1 - t0:.1f}s]", flush=True)


main()

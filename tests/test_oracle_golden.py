"""CPU: the oracle restatement is pinned to the reference's own outputs (golden vectors made
by tests/golden/make_golden.py from pyrattn) and to the reference's known-answer tests."""

import math

import numpy as np
import pytest

from helpers import GOLDEN_CASES, load_golden
from oracle import psa_oracle as orc


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    c = g["cfg"]
    lay = orc.Layout(*g["lay"])
    r = orc.run_head(g["q"], g["k"], g["v"], lay, estimator=c["estimator"], s_q=c["s_q"],
                     s_k=c["s_k"], seed=c["seed"], stride=c["stride"], mask=c["mask"],
                     thresholds=c["thresholds"], cutpoints=c["cutpoints"], tau=c["tau"],
                     sim_thresholds=c["sim_thresholds"], causal=c["causal"],
                     grid=c.get("grid"), unpermute=c.get("unpermute", False))
    # importance: same numpy ops in the same order -> identical bits
    assert np.array_equal(r["scores"], g["scores"])
    assert np.array_equal(r["mask"], g["mask"])
    if g["caps"].size:
        assert np.array_equal(r["caps"], g["caps"])
    assert np.allclose(r["out"], g["out"], rtol=0, atol=1e-12)
    fin = np.isfinite(g["lse"])
    assert np.array_equal(np.isfinite(r["lse"]), fin)
    assert np.allclose(r["lse"][fin], g["lse"][fin], rtol=0, atol=1e-12)
    assert r["skipped"] == int(g["skipped"])
    assert r["report"]["level_counts"] == g["level_counts"].tolist()
    assert r["report"]["rho_bar"] == float(g["rho_bar"])
    assert r["report"]["kv_coverage"] == float(g["kv_coverage"])
    kl, vl = r["pyramid"]
    for h in range(2, lay.levels + 1):
        if f"k_level{h}" in g:
            assert np.array_equal(kl[h - 1], g[f"k_level{h}"])
            assert np.array_equal(vl[h - 1], g[f"v_level{h}"])


@pytest.mark.parametrize("name", ["cfg1_small", "causal", "wan_b120"])
def test_materialized_equals_streaming(name):
    g = load_golden(name)
    lay = orc.Layout(*g["lay"])
    kl, vl = orc.build_pyramid(g["k"], g["v"], lay)
    o, l, s = orc.psa_materialized(g["q"], kl, vl, g["mask"], lay, g["cfg"]["causal"])
    assert np.allclose(o, g["out"], rtol=0, atol=1e-11)
    assert s == int(g["skipped"])


# ---- the reference's own known-answer tests, restated against the oracle
def test_threshold_hand_traces():
    assert orc.assign_threshold(np.array([[0.5, 0.3, 0.15, 0.05]]),
                                (0.6, 0.8, 0.95, 0.95)).tolist() == [[1, 2, 3, 0]]
    assert orc.assign_threshold(np.zeros((1, 4)), (0.5, 1.0)).tolist() == [[1, 1, 2, 2]]
    assert orc.assign_threshold(np.array([[0.05, 0.5, 0.15, 0.3]]),
                                (0.6, 0.8, 0.95, 0.95)).tolist() == [[0, 1, 3, 2]]
    assert orc.binary_mask(np.array([[0.5, 0.3, 0.15, 0.05]]), 0.85).tolist() == [[1, 1, 0, 0]]


def test_quantile_ranks_and_presets(rng):
    s = np.array([[0.1, 0.9, 0.5, 0.7, 0.3, 0.2, 0.05, 0.0]])
    assert orc.assign_quantile(s, (0.25, 0.5, 0.75, 0.75)).tolist() == [[3, 1, 2, 1, 2, 3, 0, 0]]
    exp = {"psa-1": ({1: 5, 0: 15}, 0.25, 0.25), "psa-2": ({3: 20}, 0.25, 1.0),
           "psa-3": ({1: 3, 2: 2, 3: 4, 0: 11}, 0.25, 0.45),
           "psa-4": ({1: 2, 2: 4, 3: 4, 0: 10}, 0.25, 0.5),
           "psa-5": ({1: 2, 2: 2, 3: 8, 0: 8}, 0.25, 0.6)}
    s = rng.random((4, 20))
    for name, (counts, rho, cov) in exp.items():
        m = orc.assign_quantile(s, orc.PRESETS[name])
        assert {h: int((m[0] == h).sum()) for h in np.unique(m[0])} == counts
        rep = orc.sparsity_report(m, 4)
        assert rep["rho_bar"] == rho and rep["kv_coverage"] == cov


def test_similarity_cap_and_combine(rng):
    lay = orc.Layout(32, 4, 16, 16, 2)
    row = rng.normal(size=4)
    first, second = np.tile(row, (16, 1)), np.tile(row, (16, 1))
    second[2::4] *= -1.0
    second[3::4] *= -1.0
    assert orc.level_caps(np.vstack([first, second]), lay, (0.5,)).tolist() == [2, 1]
    assert orc.combine_mask(np.array([[3, 0, 2, 1]]), np.array([2, 3, 1, 3])).tolist() == [[2, 0, 1, 1]]


def test_causal_premask_patterns():
    lay = orc.Layout(64, 8, 32, 16, 2)
    m = orc.causal_premask(np.full((2, 4), 2), lay)
    assert m.tolist() == [[1, 1, 0, 0], [2, 2, 1, 1]]


def test_pyramid_ladder_and_bias():
    lay = orc.Layout(4, 1, 4, 4, 3)
    x = np.array([[0.0], [2.0], [4.0], [6.0]])
    kl, _ = orc.build_pyramid(x, x, lay)
    assert kl[1].ravel().tolist() == [1.0, 5.0] and kl[2].ravel().tolist() == [3.0]
    assert orc.LN2 == math.log(2.0)


def test_mixed_levels_budget():
    m = np.zeros((1, 20), dtype=int)
    m[0, :3], m[0, 3:5], m[0, 5:9] = 1, 2, 3
    rep = orc.sparsity_report(m, 3)
    assert rep["rho_bar"] == 0.25 and rep["kv_coverage"] == 0.45


def test_hilbert_orders_match_reference():
    """Curve orders (permute.py:97-128): the oracle restatement and the product's host-side
    generator both equal the reference's, including the Wan 21x45x80 latent grid."""
    import paper_2512_04025_b200 as psa
    from helpers import GOLDEN_DIR
    z = np.load(GOLDEN_DIR / "hilbert_orders.npz")
    n = len([k for k in z.files if k.startswith("g")])
    for i in range(n):
        grid = tuple(int(g) for g in z[f"g{i}"])
        assert np.array_equal(orc.hilbert_order(grid), z[f"o{i}"]), grid
        p = psa.hilbert_order(grid)
        assert np.array_equal(p.order.numpy(), z[f"o{i}"]), grid
        assert np.array_equal(p.order.numpy()[p.inverse.numpy()], np.arange(len(p)))
    with pytest.raises(psa.ValidationError):
        psa.hilbert_order((6, 8))           # 2D axes must be powers of two
    with pytest.raises(psa.ValidationError):
        psa.hilbert_order((2, 2, 2, 2))
    inv = psa.invert_permutation(psa.hilbert_order((4, 4)))
    assert np.array_equal(inv.order.numpy(), psa.hilbert_order((4, 4)).inverse.numpy())

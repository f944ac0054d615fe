"""GPU parity: every sm_100a kernel against the CPU oracle on identical bf16 inputs.

Bars:
  pyramid            bit-exact == bf16_RNE(oracle fp64 pyramid)
  similarity caps    ==
  importance S       rel <= 1e-12 elementwise (fp64; exp/summation-order ulps only)
  level map / plan   bit-exact (mismatch count must be 0)
  attention O        kernel parity (oracle fed the same bf16 pyramid): rel-L2 <= 5e-3,
                     max-abs <= 1e-2 * max|ref|, lse abs <= 1e-3, skipped rows ==
                     end-to-end (oracle fp64 pyramid): rel-L2 <= 5e-3, lse abs <= 3e-2
"""

import math

import numpy as np
import pytest
import torch

from helpers import bf16_bits, bf16_round, correlated_qkv, gaussian_qkv, rel_l2, to_dev
from oracle import psa_oracle as orc

pytestmark = pytest.mark.gpu

TAUS_CFG1 = (0.164713, 0.282366, 0.376488, 0.95)


def _psa():
    import paper_2512_04025_b200 as psa
    return psa


def _bf16_levels(levels):
    return [bf16_round(x) for x in levels]


# ------------------------------------------------------------------ pyramid
@pytest.mark.parametrize("n,d,bk,H", [(4096, 64, 64, 4), (7680, 128, 120, 4), (1024, 128, 128, 8),
                                      (2048, 64, 32, 2)])
def test_pyramid_bit_exact(n, d, bk, H):
    psa = _psa()
    q, k, v = gaussian_qkv(1, 2, n, d)
    lay = psa.make_layout(n, d, bk, bk, H)
    pyr = psa.build_pyramid(to_dev(k), to_dev(v), lay)
    olay = orc.Layout(n, d, bk, bk, H)
    for h_i in range(2):
        kl, vl = orc.build_pyramid(k[h_i], v[h_i], olay)
        for h in range(2, H + 1):
            gk = pyr.level_k(h)[0, h_i].view(torch.int16).cpu().numpy()
            gv = pyr.level_v(h)[0, h_i].view(torch.int16).cpu().numpy()
            assert np.array_equal(gk, bf16_bits(kl[h - 1])), (h_i, h)
            assert np.array_equal(gv, bf16_bits(vl[h - 1])), (h_i, h)
    # reference accessor semantics: level-1 block == raw rows
    assert torch.equal(pyr.k(3, 1), to_dev(k)[0, 3 * bk:4 * bk])


def test_pyramid_flags_nonfinite():
    psa = _psa()
    lay = psa.make_layout(256, 64, 64, 64, 3)
    k = torch.randn(256, 64, device="cuda", dtype=torch.bfloat16)
    k[17, 5] = float("nan")
    with pytest.raises(psa.ValidationError):
        psa.build_pyramid(k, k.clone(), lay, check_finite=True)


# ------------------------------------------------------------------ similarity caps
@pytest.mark.parametrize("taus", [(0.7, 0.65, 0.6), (0.2, 0.1, 0.0), (-1.0, -1.0, -1.0),
                                  (1.0, 1.0, 1.0)])
def test_similarity_caps_exact(taus):
    psa = _psa()
    q, k, v = correlated_qkv(3, 2, 32, 64, 128)
    n = k.shape[1]
    lay = psa.make_layout(n, 128, 64, 64, 4)
    caps = psa.level_cap_from_similarity(to_dev(k), psa.SimThresholds(taus), layout=lay)
    olay = orc.Layout(n, 128, 64, 64, 4)
    for h in range(2):
        exp = orc.level_caps(k[h], olay, taus)
        assert np.array_equal(caps[h].cpu().numpy(), exp), h


# ------------------------------------------------------------------ importance
@pytest.mark.parametrize("n,d,bq,bk,sq,sk,red", [(4096, 64, 64, 64, 8, 8, "max"),
                                                 (7680, 128, 120, 120, 8, 8, "max"),
                                                 (2048, 128, 64, 32, 5, 7, "max"),
                                                 (4096, 64, 64, 64, 8, 8, "mean")])
def test_importance_sampled(n, d, bq, bk, sq, sk, red):
    psa = _psa()
    q, k, v = gaussian_qkv(5, 2, n, d)
    lay = psa.make_layout(n, d, bq, bk, 4 if bk % 8 == 0 else 1)
    cfg = psa.SamplerConfig(sq, sk, 0)
    s = psa.importance_sampled(to_dev(q), to_dev(k), lay, cfg, reducer=red).cpu().numpy()
    olay = orc.Layout(n, d, bq, bk, lay.levels)
    for h in range(2):
        exp = orc.importance_sampled(q[h], k[h], olay, sq, sk, 0, red)
        tol = 1e-12 if red == "max" else 1e-9
        np.testing.assert_allclose(s[h], exp, rtol=tol, atol=0)


# ------------------------------------------------------------------ level assignment
def test_assign_threshold_exact_on_oracle_scores():
    psa = _psa()
    q, k, v = gaussian_qkv(7, 3, 7680, 128)
    olay = orc.Layout(7680, 128, 120, 120, 4)
    taus = (0.1634, 0.2803, 0.3738, 0.95)
    scores = np.stack([orc.importance_sampled(q[h], k[h], olay, 8, 8, 0) for h in range(3)])
    got = psa.assign_threshold(torch.from_numpy(scores).cuda(), psa.LevelThresholds(taus))
    exp = np.stack([orc.assign_threshold(scores[h], taus) for h in range(3)])
    assert int((got.cpu().numpy() != exp).sum()) == 0


def test_assign_hand_traces():
    psa = _psa()
    t = psa.LevelThresholds((0.6, 0.8, 0.95, 0.95))
    s = torch.tensor([[0.5, 0.3, 0.15, 0.05]], dtype=torch.float64, device="cuda")
    assert psa.assign_threshold(s, t).tolist() == [[1, 2, 3, 0]]
    s2 = torch.tensor([[0.05, 0.5, 0.15, 0.3]], dtype=torch.float64, device="cuda")
    assert psa.assign_threshold(s2, t).tolist() == [[0, 1, 3, 2]]
    z = torch.zeros(1, 4, dtype=torch.float64, device="cuda")
    assert psa.assign_threshold(z, psa.LevelThresholds((0.5, 1.0))).tolist() == [[1, 1, 2, 2]]
    assert psa.binary_mask(s, 0.85).tolist() == [[1, 1, 0, 0]]
    r = torch.tensor([[0.1, 0.9, 0.5, 0.7, 0.3, 0.2, 0.05, 0.0]], dtype=torch.float64, device="cuda")
    assert psa.assign_quantile(r, psa.QuantileCutpoints((0.25, 0.5, 0.75, 0.75))).tolist() == \
        [[3, 1, 2, 1, 2, 3, 0, 0]]


def test_assign_random_rows_match_oracle(rng):
    psa = _psa()
    taus = (0.35, 0.6, 0.8, 0.92)
    s = rng.random((400, 37)) * rng.integers(0, 2, size=(400, 37))
    s[::7] *= 1e-300  # tiny magnitudes exercise the exact row total
    got = psa.assign_threshold(torch.from_numpy(s).cuda(), psa.LevelThresholds(taus)).cpu().numpy()
    assert np.array_equal(got, orc.assign_threshold(s, taus))
    for name, pts in orc.PRESETS.items():
        g = psa.assign_quantile(torch.from_numpy(s).cuda(), psa.PRESET_CUTPOINTS[name]).cpu().numpy()
        assert np.array_equal(g, orc.assign_quantile(s, pts)), name


def test_assign_low_bit_ties_match_oracle(rng):
    """Scores equal in their top 32 value bits and different below (the radix sort keys on the
    top 32 bits; the insertion pass orders these): same levels as numpy's stable argsort, also
    with exact duplicates mixed in."""
    psa = _psa()
    taus = (0.2, 0.45, 0.7, 0.9)
    base = rng.random((64, 1)) * 0.01 + 0.001
    s = base * (1.0 + rng.integers(0, 1 << 12, size=(64, 300)) * 2.0 ** -45)
    s[:, ::5] = s[:, 1::5]  # exact duplicates
    s = s[:, :300]
    rows = [s, np.concatenate([s[:, :150], rng.random((64, 150))], axis=1)]
    for x in rows:
        got = psa.assign_threshold(torch.from_numpy(x).cuda(), psa.LevelThresholds(taus))
        assert np.array_equal(got.cpu().numpy(), orc.assign_threshold(x, taus))


# ------------------------------------------------------------------ attention kernel
def _attention_case(q, k, v, mask, lay_args, causal=False, check_e2e=True):
    psa = _psa()
    n, d, bq, bk, H = lay_args
    lay = psa.make_layout(*lay_args)
    olay = orc.Layout(*lay_args)
    heads = q.shape[0]
    pyr = psa.build_pyramid(to_dev(k), to_dev(v), lay)
    res = psa.psa_streaming(to_dev(q), pyr, torch.from_numpy(mask).cuda(), causal=causal)
    out = res.out.float().cpu().numpy().astype(np.float64)
    lse = res.row_log_normalizers.cpu().numpy().astype(np.float64)
    skipped_exp = 0
    for h in range(heads):
        kl, vl = orc.build_pyramid(k[h], v[h], olay)
        ref_o, ref_l, sk = orc.psa_materialized(q[h], _bf16_levels(kl), _bf16_levels(vl),
                                                mask[h], olay, causal)
        skipped_exp += sk
        assert rel_l2(out[h], ref_o) <= 5e-3
        assert float(np.abs(out[h] - ref_o).max()) <= 1e-2 * max(float(np.abs(ref_o).max()), 1e-30)
        fin = np.isfinite(ref_l)
        assert np.array_equal(np.isfinite(lse[h]), fin)
        if fin.any():
            assert float(np.abs(lse[h][fin] - ref_l[fin]).max()) <= 1e-3
        if check_e2e:
            e_o, e_l, _ = orc.psa_streaming(q[h], kl, vl, mask[h], olay, causal)
            assert rel_l2(out[h], e_o) <= 5e-3
            if fin.any():
                assert float(np.abs(lse[h][fin] - e_l[fin]).max()) <= 3e-2
    assert res.skipped_rows == skipped_exp
    return res


@pytest.mark.parametrize("n,d,b,H", [(1024, 64, 64, 4), (1920, 128, 120, 4), (1024, 128, 128, 4),
                                     (512, 128, 32, 3)])
def test_attention_random_masks(n, d, b, H, rng):
    q, k, v = gaussian_qkv(11, 2, n, d)
    nb = n // b
    mask = rng.integers(0, H + 1, size=(2, nb, nb))
    mask[0, 0, :] = 0          # an entirely skipped query block
    mask[1, 1, :] = 0
    mask[1, 1, 2] = 1
    _attention_case(q, k, v, mask, (n, d, b, b, H))


def test_attention_dense_equals_full_attention():
    psa = _psa()
    q, k, v = gaussian_qkv(13, 1, 1024, 128)
    res = psa.full_attention(to_dev(q[0]), to_dev(k[0]), to_dev(v[0]))
    ref, lse = orc.full_attention(q[0], k[0], v[0])
    assert rel_l2(res.out.float().cpu().numpy(), ref) <= 5e-3
    assert float(np.abs(res.row_log_normalizers.cpu().numpy() - lse).max()) <= 1e-3


def test_attention_causal_full():
    psa = _psa()
    q, k, v = gaussian_qkv(17, 1, 1024, 64)
    res = psa.causal_full_attention(to_dev(q[0]), to_dev(k[0]), to_dev(v[0]))
    ref, lse = orc.causal_full_attention(q[0], k[0], v[0])
    assert rel_l2(res.out.float().cpu().numpy(), ref) <= 5e-3
    assert float(np.abs(res.row_log_normalizers.cpu().numpy() - lse).max()) <= 1e-3


def test_attention_causal_pyramid(rng):
    q, k, v = gaussian_qkv(19, 2, 2048, 128)
    lay = orc.Layout(2048, 128, 64, 64, 4)
    m = rng.integers(0, 5, size=(2, 32, 32))
    m = np.stack([orc.causal_premask(m[h], lay) for h in range(2)])
    _attention_case(q, k, v, m, (2048, 128, 64, 64, 4), causal=True)


def test_attention_duplicated_tokens_level_bias():
    """Duplicated K/V rows: pooling is lossless, so level h must equal level 1 (the (h-1) ln 2
    bias restores the pooled mass exactly) — attention.py docstring, test_attention.py:138-146."""
    psa = _psa()
    rng = np.random.default_rng(23)
    n, d = 1024, 128
    q = bf16_round(rng.standard_normal((1, n, d)))
    base = bf16_round(rng.standard_normal((1, n // 4, d)))
    k = np.repeat(base, 4, axis=1)
    v = np.repeat(bf16_round(rng.standard_normal((1, n // 4, d))), 4, axis=1)
    lay = psa.make_layout(n, d, 128, 128, 3)
    pyr = psa.build_pyramid(to_dev(k), to_dev(v), lay)
    outs = []
    for h in (1, 2, 3):
        m = torch.full((1, 8, 8), h, dtype=torch.int64, device="cuda")
        outs.append(psa.psa_streaming(to_dev(q), pyr, m).out.float().cpu().numpy())
    assert rel_l2(outs[1], outs[0]) <= 5e-3
    assert rel_l2(outs[2], outs[0]) <= 5e-3


def test_mask_validation():
    psa = _psa()
    lay = psa.make_layout(256, 64, 64, 64, 2)
    q = torch.randn(256, 64, device="cuda", dtype=torch.bfloat16)
    pyr = psa.build_pyramid(q, q, lay)
    with pytest.raises(psa.ValidationError):
        psa.psa_streaming(q, pyr, torch.full((4, 4), 3, device="cuda"))
    with pytest.raises(psa.ValidationError):  # pooled level on a straddling pair
        psa.psa_streaming(q, pyr, torch.full((4, 4), 2, device="cuda"), causal=True)
    # host Q is staged onto the device like any array-like (linalg.py:15-24), same result
    m1 = torch.ones(4, 4, device="cuda", dtype=torch.int64)
    assert torch.equal(psa.psa_streaming(q.cpu(), pyr, m1).out, psa.psa_streaming(q, pyr, m1).out)
    with pytest.raises(psa.ValidationError):  # non-numeric input
        psa.psa_streaming([["a"] * 64] * 256, pyr, m1)


# ------------------------------------------------------------------ fused pipeline
@pytest.mark.parametrize("case", ["cfg1", "wan_small", "quantile", "binary", "simcap", "causal_gqa",
                                  "mean", "antidiag_gqa_causal", "antidiag_wan",
                                  "grid_causal_gqa"])
def test_pipeline_level_map_and_output(case):
    psa = _psa()
    kw = dict(estimator="sampled-max", s_q=8, s_k=8, seed=0, mask="threshold",
              thresholds=TAUS_CFG1)
    hq = hkv = 2
    if case == "cfg1":
        n, d, b, H = 4096, 64, 64, 4
    elif case == "wan_small":
        n, d, b, H = 7680, 128, 120, 4
        kw["thresholds"] = (0.1634, 0.2803, 0.3738, 0.95)
    elif case == "quantile":
        n, d, b, H = 4096, 128, 64, 4
        kw.update(mask="psa-3", thresholds=None)
    elif case == "binary":
        n, d, b, H = 4096, 128, 128, 4
        kw.update(mask="binary", tau=0.5, thresholds=None)
    elif case == "simcap":
        n, d, b, H = 2048, 128, 64, 4
        kw["sim_thresholds"] = (0.7, 0.65, 0.6)
    elif case == "causal_gqa":
        n, d, b, H = 2048, 128, 64, 4
        kw["causal"] = True
        hq, hkv = 4, 2
    elif case == "antidiag_gqa_causal":  # cfg4 recipe at reduced size
        n, d, b, H = 4096, 128, 64, 4
        kw.update(estimator="antidiagonal", stride=8, causal=True, sim_thresholds=(0.75, 0.7, 0.7))
        hq, hkv = 4, 2
    elif case == "antidiag_wan":
        n, d, b, H = 3840, 128, 120, 4
        kw.update(estimator="antidiagonal", stride=8, thresholds=(0.1634, 0.2803, 0.3738, 0.95))
    elif case == "grid_causal_gqa":  # curve permutation (fused gathers / scatter) + causal + GQA
        n, d, b, H = 2048, 128, 64, 4
        kw.update(causal=True, grid=(8, 16, 16), unpermute=True)
        hq, hkv = 4, 2
    else:
        n, d, b, H = 4096, 64, 64, 4
        kw["estimator"] = "sampled-mean"
    if case == "simcap":
        q, k, v = correlated_qkv(29, 2, 32, 64, d)
    else:
        q, k, v = gaussian_qkv(29, hq, n, d, hkv)
    res = psa.psa_attention(to_dev(q), to_dev(k), to_dev(v), b_q=b, b_k=b, levels=H,
                            tile_len=128, **kw)
    lm = res.level_map.cpu().numpy()[0]
    lay = orc.Layout(n, d, b, b, H)
    okw = {x: kw.get(x) for x in ("estimator", "s_q", "s_k", "seed", "mask", "thresholds",
                                  "cutpoints", "tau", "sim_thresholds", "causal", "stride",
                                  "grid")}
    okw["unpermute"] = bool(kw.get("unpermute", False))
    out = res.out.float().cpu().numpy()
    mism = 0
    for h in range(hq):
        hk = h // (hq // hkv)
        r = orc.run_head(q[h], k[hk], v[hk], lay, executor="materialized", **okw)
        mism += int((lm[h] != r["mask"]).sum())
        assert rel_l2(out[h], r["out"]) <= 5e-3, h
    assert mism == 0


# ------------------------------------------------------------------ host staging (e2e API)
@pytest.mark.parametrize("hq,hkv,causal,per_group,batch", [
    (6, 6, False, 2, 1), (8, 2, True, 1, 1), (3, 3, False, None, 1), (4, 2, False, None, 2)])
def test_staged_host_path_bit_identical(hq, hkv, causal, per_group, batch):
    """psa_attention on host tensors (pipelined H2D/compute/D2H over head groups) returns exactly
    the device path's O, lse, level map and counts."""
    psa = _psa()
    n, d, b = 2048, 128, 64
    q, k, v = gaussian_qkv(11, hq * batch, n, d, kv_heads=hkv * batch)
    qh, kh, vh = (torch.from_numpy(x).to(torch.bfloat16).reshape(batch, -1, n, d)
                  for x in (q, k, v))
    kw = dict(b_q=b, b_k=b, levels=4, estimator="sampled-max", s_q=8, s_k=8, seed=0,
              mask="threshold", thresholds=TAUS_CFG1, causal=causal)
    dev = psa.psa_attention(qh.cuda(), kh.cuda(), vh.cuda(), **kw)
    torch.cuda.synchronize()
    host = psa.psa_attention(qh.pin_memory(), kh.pin_memory(), vh.pin_memory(),
                             kv_heads_per_group=per_group, keep_level_map=True, **kw)
    assert not host.out.is_cuda and host.out.shape == qh.shape
    assert torch.equal(host.out.view(torch.int16), dev.out.cpu().view(torch.int16))
    assert torch.equal(host.lse, dev.lse.cpu())
    assert torch.equal(host.level_map, dev.level_map.cpu())
    assert host.level_counts == dev.plan.level_counts.cpu().tolist()
    assert host.skipped_rows() == dev.skipped_rows()
    assert host.sparsity().rho_bar == dev.sparsity().rho_bar


# ------------------------------------------------------------------ exact int8-sliced logits
def _with_tiny(x, rng, rows, per_row):
    """Scale `per_row` random entries of the given rows by 2^-20 (elements below the int8 slice
    grid: exercises the exact tiny-element correction, or the fp64 fallback past 4 per row)."""
    x = x.copy()
    for r in rows:
        cols = rng.choice(x.shape[-1], per_row, replace=False)
        x[..., r, cols] *= 2.0 ** -20
    return bf16_round(x)


@pytest.mark.parametrize("kind,n,d,b,sk_or_stride", [
    ("sampled", 4096, 128, 64, 8), ("sampled", 3840, 128, 120, 8), ("sampled", 2048, 64, 64, 7),
    ("antidiag", 4096, 128, 64, 8), ("antidiag", 3840, 128, 120, 4), ("antidiag", 1920, 64, 120, 8)])
@pytest.mark.parametrize("tiny", [0, 2, 6, -1])
def test_int8_exact_logits_match_fp64_path(kind, n, d, b, sk_or_stride, tiny):
    _int8_vs_fp64(kind, n, d, b, sk_or_stride, tiny)


@pytest.mark.parametrize("kind,n,d,b,sk_or_stride", [
    ("sampled", 12288, 64, 64, 8), ("antidiag", 12288, 64, 64, 8)])
@pytest.mark.parametrize("tiny", [0, 6])
def test_int8_key_split_merge(kind, n, d, b, sk_or_stride, tiny):
    """Sizes whose key tiles are split over several CTAs (xl_merge_kernel combines the per-split
    (m, l)); with tiny=6 one head is flagged and left to the fp64 kernel by the merge."""
    _int8_vs_fp64(kind, n, d, b, sk_or_stride, tiny)


def _int8_vs_fp64(kind, n, d, b, sk_or_stride, tiny):
    """The int8 tensor-core logits (psa_xlogits.cu) reproduce the fp64 DMMA path: scores agree to
    a few ulps (only the softmax-denominator summation order differs), level maps exactly, and
    both match the oracle at 1e-12. tiny=2: exact corrections; tiny=6: fp64 fallback heads;
    tiny=-1: one head with 32x larger queries (logits up to ~100: peaked softmax rows)."""
    from paper_2512_04025_b200.importance import antidiagonal_scores, importance_scores
    from paper_2512_04025_b200.mask import assign_levels_device
    psa = _psa()
    rng = np.random.default_rng(17 + tiny)
    q, k, v = gaussian_qkv(23, 3, n, d)
    if tiny < 0:
        q[1] = q[1] * 32.0  # power of two: still exact bf16
    elif tiny:
        q[1] = _with_tiny(q[1], rng, rng.choice(n, 64, replace=False), tiny)
        k[2] = _with_tiny(k[2], rng, rng.choice(n, 64, replace=False), tiny)
    lay = psa.make_layout(n, d, b, b, 4)
    q4, k4 = to_dev(q)[None], to_dev(k)[None]
    if kind == "sampled":
        cfg = psa.SamplerConfig(8, sk_or_stride, 0)
        fast = importance_scores(q4, k4, lay, cfg, "max")
        slow = importance_scores(q4, k4, lay, cfg, "max", fp64_only=True)
    else:
        fast = antidiagonal_scores(q4, k4, lay, sk_or_stride)
        slow = antidiagonal_scores(q4, k4, lay, sk_or_stride, fp64_only=True)
    np.testing.assert_allclose(fast.cpu().numpy(), slow.cpu().numpy(), rtol=1e-14, atol=0)
    rule = psa.LevelThresholds(TAUS_CFG1)
    pf = assign_levels_device(fast, mode="threshold", rule=rule, levels=4, b_q=b, b_k=b, hkv=3)
    ps = assign_levels_device(slow, mode="threshold", rule=rule, levels=4, b_q=b, b_k=b, hkv=3)
    assert torch.equal(pf.level_map, ps.level_map)
    olay = orc.Layout(n, d, b, b, 4)
    f = fast.cpu().numpy()[0]
    for h in range(3):
        exp = (orc.importance_sampled(q[h], k[h], olay, 8, sk_or_stride, 0, "max")
               if kind == "sampled" else orc.importance_antidiagonal(q[h], k[h], olay, sk_or_stride))
        np.testing.assert_allclose(f[h], exp, rtol=1e-12, atol=0)


# ------------------------------------------------------------------ token permutation
@pytest.mark.parametrize("grid,d", [((32, 32), 64), ((6, 10, 16), 128), ((21, 45, 8), 128)])
def test_apply_permutation_exact(grid, d):
    """psa_gather_rows == numpy fancy indexing (permute.py:131-137), bit for bit; the inverse
    permutation restores the input."""
    psa = _psa()
    n = int(np.prod(grid))
    x = torch.randn(2, 3, n, d, dtype=torch.bfloat16, device="cuda")
    p = psa.hilbert_order(grid)
    y = psa.apply_permutation(x, p)
    ref = x.cpu()[:, :, p.order]
    assert torch.equal(y.cpu().view(torch.int16), ref.view(torch.int16))
    back = psa.apply_permutation(y, psa.invert_permutation(p))
    assert torch.equal(back.view(torch.int16), x.view(torch.int16))
    single = psa.apply_permutation(x[0, 0], p)  # (n, d) form
    assert torch.equal(single.cpu().view(torch.int16), ref[0, 0].view(torch.int16))


@pytest.mark.parametrize("grid,d,b,levels", [((16, 16, 16), 128, 64, 4), ((21, 45, 8), 128, 120, 4),
                                             ((32, 32), 64, 64, 1), ((6, 10, 16), 128, 96, 3)])
def test_fused_permutation_pyramid_and_scatter(grid, d, b, levels):
    """The permutation fused into the pyramid loads (psa_pyramid_build_gather) equals gather then
    build_pyramid bit for bit (level 1 = the permuted K/V); the attention epilogue's scatter
    (psa_attn_fwd_scatter) equals attention then the inverse gather, bit for bit."""
    from paper_2512_04025_b200.attention import attention_forward
    from paper_2512_04025_b200.mask import plan_from_mask
    from paper_2512_04025_b200.pyramid import build_pyramid_gather
    psa = _psa()
    n = int(np.prod(grid))
    torch.manual_seed(3)
    q, k, v = (torch.randn(1, 2, n, d, dtype=torch.bfloat16, device="cuda") for _ in range(3))
    lay = psa.make_layout(n, d, b, b, levels)
    p = psa.hilbert_order(grid)
    order, inverse = p.on(q.device)
    fused = build_pyramid_gather(k, v, lay, order)
    kg, vg = psa.apply_permutation(k, p), psa.apply_permutation(v, p)
    plain = psa.build_pyramid(kg, vg, lay)
    bits = lambda t: t.view(torch.int16)  # noqa: E731
    assert torch.equal(bits(fused.k_raw), bits(kg)) and torch.equal(bits(fused.v_raw), bits(vg))
    if levels > 1:
        assert torch.equal(bits(fused.k_pyr), bits(plain.k_pyr))
        assert torch.equal(bits(fused.v_pyr), bits(plain.v_pyr))
    qg = psa.apply_permutation(q, p)
    rng = np.random.default_rng(5)
    mask = torch.from_numpy(rng.integers(0, levels + 1, size=(1, 2, lay.n_q, lay.n_k))).cuda()
    plan = plan_from_mask(mask, lay, False, 1, 2)
    out, lse, _ = attention_forward(qg, plain, plan, False)
    out_s, lse_s, _ = attention_forward(qg, fused, plan, False, out_rows=order)
    assert torch.equal(bits(out_s), bits(psa.apply_permutation(out, psa.invert_permutation(p))))
    assert torch.equal(lse_s, lse[:, :, inverse])


# ------------------------------------------------------------------ block-tile schedule API
@pytest.mark.parametrize("causal", [False, True])
def test_execute_schedule_equals_streaming(causal, rng):
    """execute_schedule (scheduler.py:203-269) on the GPU executor == psa_streaming on the same
    mask (tiling only re-chunks the online softmax), and matches the oracle."""
    psa = _psa()
    n, d, b, H = 2048, 128, 64, 4
    q, k, v = gaussian_qkv(41, 1, n, d)
    lay = psa.make_layout(n, d, b, b, H)
    m = rng.integers(0, H + 1, size=(lay.n_q, lay.n_k))
    olay = orc.Layout(n, d, b, b, H)
    if causal:
        m = orc.causal_premask(m, olay)
    pyr = psa.build_pyramid(to_dev(k[0]), to_dev(v[0]), lay)
    sch = psa.build_schedule(m, lay, 128)
    a = psa.execute_schedule(to_dev(q[0]), pyr, sch, causal=causal)
    s = psa.psa_streaming(to_dev(q[0]), pyr, torch.from_numpy(m).cuda(), causal=causal)
    assert torch.equal(a.out.view(torch.int16), s.out.view(torch.int16))
    assert a.skipped_rows == s.skipped_rows
    kl, vl = orc.build_pyramid(k[0], v[0], olay)
    o, l, sk = orc.psa_streaming(q[0], kl, vl, m, olay, causal)
    assert rel_l2(a.out.float().cpu().numpy(), o) <= 5e-3
    assert psa.utilization(sch).utilization <= 1.0


def test_plan_utilization_counts_executed_tiles():
    psa = _psa()
    n, d, b = 3840, 128, 120
    q, k, v = gaussian_qkv(43, 2, n, d)
    res = psa.psa_attention(to_dev(q), to_dev(k), to_dev(v), b_q=b, b_k=b, levels=4,
                            estimator="sampled-max", s_q=8, s_k=8, seed=0, mask="threshold",
                            thresholds=(0.1634, 0.2803, 0.3738, 0.95))
    lay = psa.make_layout(n, d, b, b, 4)
    u = psa.plan_utilization(res.plan, lay)
    counts = res.plan.level_counts.cpu().tolist()
    assert u.useful_rows == sum(c * (b >> (h - 1)) for h, c in enumerate(counts) if h)
    assert 0.5 < u.utilization <= 1.0


# ------------------------------------------------------------------ more layouts (round 2)
# b_q != b_k for the sampled estimator, a b_q that is not a power of two, deep pyramids (6 and
# 8 levels: level-8 blocks pool to one row), d = 64 with the antidiagonal estimator under causal
# GQA, and batch 2 -- each against the oracle's stage order (level map ==, O within the bar).
EXTRA = {
    "bq128_bk64_sampled": dict(n=4096, d=128, b_q=128, b_k=64, levels=4, hq=2, hkv=2,
                               kw=dict(estimator="sampled-max", s_q=8, s_k=8, seed=1,
                                       mask="threshold", thresholds=TAUS_CFG1)),
    "bq90_bk64": dict(n=5760, d=128, b_q=90, b_k=64, levels=4, hq=2, hkv=1,
                      kw=dict(estimator="sampled-max", s_q=8, s_k=8, seed=2, mask="threshold",
                              thresholds=TAUS_CFG1)),
    "levels6_b96_d64": dict(n=3072, d=64, b_q=96, b_k=96, levels=6, hq=2, hkv=2,
                            kw=dict(estimator="sampled-max", s_q=8, s_k=8, seed=3, mask="threshold",
                                    thresholds=(0.12, 0.2, 0.28, 0.36, 0.45, 0.95))),
    "levels8_b128": dict(n=4096, d=128, b_q=128, b_k=128, levels=8, hq=2, hkv=2,
                         kw=dict(estimator="sampled-max", s_q=8, s_k=8, seed=4, mask="threshold",
                                 thresholds=(0.1, 0.16, 0.22, 0.28, 0.34, 0.4, 0.5, 0.95))),
    "antidiag_d64_causal_gqa": dict(n=4096, d=64, b_q=64, b_k=32, levels=4, hq=6, hkv=2,
                                    kw=dict(estimator="antidiagonal", stride=4, mask="threshold",
                                            thresholds=TAUS_CFG1, causal=True)),
    "batch2_causal": dict(n=2048, d=128, b_q=64, b_k=64, levels=4, hq=2, hkv=2, batch=2,
                          kw=dict(estimator="sampled-max", s_q=8, s_k=8, seed=5, mask="threshold",
                                  thresholds=TAUS_CFG1, causal=True)),
}


@pytest.mark.parametrize("case", sorted(EXTRA))
def test_pipeline_more_layouts(case):
    psa = _psa()
    c = EXTRA[case]
    n, d, hq, hkv, batch = c["n"], c["d"], c["hq"], c["hkv"], c.get("batch", 1)
    qs, ks, vs = zip(*(gaussian_qkv(41 + bi, hq, n, d, hkv) for bi in range(batch)))
    q4, k4, v4 = (torch.stack([to_dev(x) for x in xs]) for xs in (qs, ks, vs))
    res = psa.psa_attention(q4, k4, v4, b_q=c["b_q"], b_k=c["b_k"], levels=c["levels"],
                            tile_len=128, **c["kw"])
    lm = res.level_map.cpu().numpy()
    out = res.out.float().cpu().numpy()
    lay = orc.Layout(n, d, c["b_q"], c["b_k"], c["levels"])
    okw = {x: c["kw"].get(x) for x in ("estimator", "s_q", "s_k", "seed", "mask", "thresholds",
                                       "stride", "causal")}
    okw["causal"] = bool(okw["causal"])
    mism = 0
    for bi in range(batch):
        for h in range(hq):
            hk = h // (hq // hkv)
            r = orc.run_head(qs[bi][h], ks[bi][hk], vs[bi][hk], lay, executor="materialized",
                             **okw)
            mism += int((lm[bi, h] != r["mask"]).sum())
            assert rel_l2(out[bi, h], r["out"]) <= 5e-3, (bi, h)
    assert mism == 0

"""Backward of the multi-level attention (psa_backward.cu) against the autograd of the forward's
definition in fp64 (attention.py:171-218 and blocks.py:93-109 restated in torch with the mask held
fixed). The reference package has no backward, so this torch fp64 restatement is the
oracle for a floating-point kernel. Bar: relative L2 error <= 1e-2 per gradient (bf16 inputs,
bf16 pooled levels and bf16 MMA operands on the GPU, fp64 in the oracle)."""

import math

import numpy as np
import pytest
import torch

from helpers import gaussian_qkv, rel_l2, to_dev

pytestmark = pytest.mark.gpu


def _oracle(q, k, v, lm, b_q, b_k, causal):
    """fp64 forward with autograd: q [Hq, n, d], k/v [Hkv, n, d], lm int [Hq, n_q, n_k]."""
    Hq, n, d = q.shape
    grp = Hq // k.shape[0]
    scale = 1.0 / math.sqrt(d)
    heads = []
    for hq in range(Hq):
        hk = hq // grp
        rows = []
        for i in range(n // b_q):
            qi = q[hq, i * b_q:(i + 1) * b_q]
            ks, vs, bias, masks = [], [], [], []
            qpos = torch.arange(i * b_q, (i + 1) * b_q)
            for j in range(n // b_k):
                h = int(lm[hq, i, j])
                if h == 0:
                    continue
                f = 2 ** (h - 1)
                kp = k[hk, j * b_k:(j + 1) * b_k].reshape(b_k // f, f, d).mean(1)
                vp = v[hk, j * b_k:(j + 1) * b_k].reshape(b_k // f, f, d).mean(1)
                ks.append(kp)
                vs.append(vp)
                bias.append(torch.full((b_k // f,), (h - 1) * math.log(2.0), dtype=q.dtype))
                straddle = causal and (j + 1) * b_k - 1 > i * b_q
                kpos = torch.arange(j * b_k, (j + 1) * b_k, f)
                masks.append((kpos[None, :] > qpos[:, None]) if straddle
                             else torch.zeros(b_q, b_k // f, dtype=torch.bool))
            if not ks:
                rows.append(torch.zeros(b_q, d, dtype=q.dtype))
                continue
            s = qi @ torch.cat(ks).T * scale + torch.cat(bias)
            s = s.masked_fill(torch.cat(masks, dim=1), -math.inf)
            dead = torch.isinf(s).all(dim=1, keepdim=True)
            p = torch.softmax(s.masked_fill(dead, 0.0), dim=1).masked_fill(dead, 0.0)
            rows.append(p @ torch.cat(vs))
        heads.append(torch.cat(rows))
    return torch.stack(heads)


@pytest.mark.parametrize("n,d,b_q,b_k,hq,hkv,causal", [
    (1024, 64, 64, 64, 2, 2, False), (960, 128, 120, 120, 2, 1, False),
    (1024, 128, 128, 64, 4, 2, True), (512, 64, 64, 64, 3, 3, True),
    # b_q % 4 != 0: lse / D rows staged by the producer warp instead of a bulk copy
    (720, 128, 90, 120, 2, 2, False),
    # n_k = 9: the last packed dK/dV unit of levels 2-4 holds fewer than 2^(h-1) blocks
    (1152, 128, 128, 128, 2, 1, False)])
def test_backward_matches_fp64_autograd(n, d, b_q, b_k, hq, hkv, causal):
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.attention import attention_backward
    q, k, v = gaussian_qkv(61, hq, n, d, hkv)
    rng = np.random.default_rng(62)
    g = rng.standard_normal((hq, n, d))
    cfg = psa.RunConfig.from_dict(dict(n=n, d=d, b_q=b_q, b_k=b_k, levels=4,
                                       estimator="sampled-max", s_q=8, s_k=8, seed=0,
                                       mask="threshold", thresholds=[0.25, 0.45, 0.6, 0.9],
                                       tile_len=128, causal=causal))
    q4, k4, v4 = (to_dev(x)[None] for x in (q, k, v))
    res = psa.psa_forward_4d(q4, k4, v4, cfg)
    lm = res.plan.level_map[0].cpu().numpy()
    assert (lm > 1).any() and (lm == 1).any()  # several levels exercised
    dq, dk, dv = attention_backward(q4, res.pyramid, res.plan, causal, res.out, res.lse,
                                    to_dev(g)[None])
    qt, kt, vt = (torch.from_numpy(x).requires_grad_(True) for x in (q, k, v))
    out = _oracle(qt, kt, vt, lm, b_q, b_k, causal)
    assert rel_l2(res.out[0].float().cpu().numpy(), out.detach().numpy()) <= 1e-2
    (out * torch.from_numpy(g)).sum().backward()
    for mine, ref in ((dq, qt.grad), (dk, kt.grad), (dv, vt.grad)):
        assert rel_l2(mine[0].float().cpu().numpy(), ref.numpy()) <= 1e-2


def test_autograd_function_matches_direct_backward():
    """psa_attention_differentiable: loss.backward() gives the kernels' gradients on the user's
    tensors (through the bf16 cast) and lse carries no gradient."""
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.attention import attention_backward
    q, k, v = gaussian_qkv(63, 2, 1024, 64)
    qd, kd, vd = (torch.from_numpy(x).float().cuda().requires_grad_(True) for x in (q, k, v))
    kw = dict(b_q=64, b_k=64, levels=4, estimator="sampled-max", s_q=8, s_k=8, seed=0,
              mask="threshold", thresholds=[0.25, 0.45, 0.6, 0.9], tile_len=128)
    out, lse = psa.psa_attention_differentiable(qd, kd, vd, **kw)
    assert out.shape == (2, 1024, 64) and not lse.requires_grad
    g = torch.randn_like(out)
    (out.float() * g).sum().backward()
    cfg = psa.RunConfig.from_dict(dict(n=1024, d=64, **kw))
    q4, k4, v4 = (x.detach().to(torch.bfloat16)[None] for x in (qd, kd, vd))
    res = psa.psa_forward_4d(q4, k4, v4, cfg)
    dq, dk, dv = attention_backward(q4, res.pyramid, res.plan, False, res.out, res.lse,
                                    g.to(torch.bfloat16)[None])
    for mine, ref in ((qd.grad, dq), (kd.grad, dk), (vd.grad, dv)):
        assert torch.equal(mine.to(torch.bfloat16), ref[0])


@pytest.mark.parametrize("B,levels,taus", [
    (2, 4, (0.25, 0.45, 0.6, 0.9)),
    # deep pyramids: level-6..8 dK/dV units hold 16 of the 2^(h-1) blocks (per-entry 16-bit mask)
    (1, 6, (0.1, 0.2, 0.3, 0.4, 0.5, 0.95)),
    (1, 8, (0.08, 0.16, 0.24, 0.32, 0.4, 0.5, 0.6, 0.95))])
def test_backward_batch_and_deep_levels(B, levels, taus):
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.attention import attention_backward
    n, d, b, hq, hkv = 4096, 128, 128, 2, 1
    qs, ks, vs = zip(*(gaussian_qkv(70 + bi, hq, n, d, hkv) for bi in range(B)))
    q, k, v = (np.stack(x) for x in (qs, ks, vs))
    g = np.random.default_rng(71).standard_normal((B, hq, n, d))
    cfg = psa.RunConfig.from_dict(dict(n=n, d=d, b_q=b, b_k=b, levels=levels,
                                       estimator="sampled-max", s_q=8, s_k=8, seed=0,
                                       mask="threshold", thresholds=list(taus), tile_len=128))
    q4, k4, v4 = (to_dev(x) for x in (q, k, v))
    res = psa.psa_forward_4d(q4, k4, v4, cfg)
    lm = res.plan.level_map.cpu().numpy()
    assert (lm == levels).any() and (lm == 1).any()
    dq, dk, dv = attention_backward(q4, res.pyramid, res.plan, False, res.out, res.lse, to_dev(g))
    for bi in range(B):
        qt, kt, vt = (torch.from_numpy(x[bi]).requires_grad_(True) for x in (q, k, v))
        out = _oracle(qt, kt, vt, lm[bi], b, b, False)
        assert rel_l2(res.out[bi].float().cpu().numpy(), out.detach().numpy()) <= 1e-2
        (out * torch.from_numpy(g[bi])).sum().backward()
        for mine, ref in ((dq, qt.grad), (dk, kt.grad), (dv, vt.grad)):
            assert rel_l2(mine[bi].float().cpu().numpy(), ref.numpy()) <= 1e-2, (bi, levels)


def test_autograd_causal_gqa_matches_fp64():
    """psa_attention_differentiable with causal GQA (4 query heads on 2 KV heads): gradients on
    the user's tensors against the fp64 autograd oracle with the same level map."""
    import paper_2512_04025_b200 as psa
    n, d, b_q, b_k, hq, hkv = 1024, 128, 128, 64, 4, 2
    q, k, v = gaussian_qkv(73, hq, n, d, hkv)
    g = np.random.default_rng(74).standard_normal((hq, n, d))
    kw = dict(b_q=b_q, b_k=b_k, levels=4, estimator="sampled-max", s_q=8, s_k=8, seed=0,
              mask="threshold", thresholds=[0.25, 0.45, 0.6, 0.9], tile_len=128, causal=True)
    qd, kd, vd = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    out, _ = psa.psa_attention_differentiable(qd, kd, vd, **kw)
    (out.float() * torch.from_numpy(g).float().cuda()).sum().backward()
    cfg = psa.RunConfig.from_dict(dict(n=n, d=d, **kw))
    res = psa.psa_forward_4d(*(x.detach()[None] for x in (qd, kd, vd)), cfg)
    lm = res.plan.level_map[0].cpu().numpy()
    qt, kt, vt = (torch.from_numpy(x).requires_grad_(True) for x in (q, k, v))
    ref = _oracle(qt, kt, vt, lm, b_q, b_k, True)
    (ref * torch.from_numpy(g)).sum().backward()
    for mine, r in ((qd.grad, qt.grad), (kd.grad, kt.grad), (vd.grad, vt.grad)):
        assert rel_l2(mine.float().cpu().numpy(), r.numpy()) <= 1e-2
    # an in-place edit of K between forward and backward is caught by autograd
    out2, _ = psa.psa_attention_differentiable(qd, kd, vd, **kw)
    with torch.no_grad():
        kd.add_(0)
    with pytest.raises(RuntimeError):
        out2.float().sum().backward()

"""GPU: the drop-in boundary accepts what the reference accepts and rejects what it rejects.
pkg/src/pyrattn/linalg.py:15-24 (as_matrix): array-likes are converted, non-finite entries raise
ValidationError; the GPU entry points stage host / numpy inputs onto the device (the compute is
always the sm_100a kernels) and raise the same error class on NaN / Inf."""

import numpy as np
import pytest
import torch

from helpers import gaussian_qkv, to_dev

pytestmark = pytest.mark.gpu

KW = dict(b_q=64, b_k=64, levels=4, estimator="sampled-max", s_q=8, s_k=8, seed=0,
          mask="threshold", thresholds=[0.16, 0.28, 0.37, 0.95], tile_len=128)


def test_numpy_inputs_match_device_inputs():
    import paper_2512_04025_b200 as psa
    q, k, v = gaussian_qkv(31, 1, 1024, 64)
    lay = psa.make_layout(1024, 64, 64, 64, 4)
    cfg = psa.SamplerConfig(8, 8, 0)
    s_np = psa.importance_sampled(q[0], k[0], lay, cfg)
    s_dev = psa.importance_sampled(to_dev(q[0]), to_dev(k[0]), lay, cfg)
    assert torch.equal(s_np, s_dev)
    pyr_np = psa.build_pyramid(k[0], v[0], lay)
    pyr = psa.build_pyramid(to_dev(k[0]), to_dev(v[0]), lay)
    assert torch.equal(pyr_np.level_k(3), pyr.level_k(3))
    m = psa.assign_threshold(s_np.cpu().numpy(), psa.LevelThresholds(KW["thresholds"]))
    out_np = psa.psa_streaming(q[0], pyr, m.cpu().numpy())
    out_dev = psa.psa_streaming(to_dev(q[0]), pyr, m)
    assert torch.equal(out_np.out, out_dev.out)
    caps = psa.level_cap_from_similarity(k[0], psa.SimThresholds((0.7, 0.65, 0.6)), layout=lay)
    assert torch.equal(psa.combine_mask(m.cpu().numpy(), caps.cpu().numpy()),
                       psa.combine_mask(m, caps))
    res = psa.psa_attention(q, k, v, **KW)  # numpy (heads, n, d): staged like host tensors
    ref = psa.psa_attention(to_dev(q), to_dev(k), to_dev(v), **KW)
    assert torch.equal(res.out, ref.out.cpu())


@pytest.mark.parametrize("where", ["q", "k", "v"])
def test_nonfinite_inputs_raise(where):
    import paper_2512_04025_b200 as psa
    q, k, v = (to_dev(x) for x in gaussian_qkv(33, 2, 1024, 64))
    x = {"q": q, "k": k, "v": v}[where]
    x[1, 100, 7] = float("nan") if where != "v" else float("inf")
    with pytest.raises(psa.ValidationError):
        psa.psa_attention(q, k, v, **KW)
    with pytest.raises(psa.ValidationError):  # host tensors: staged path
        psa.psa_attention(q.cpu(), k.cpu(), v.cpu(), **KW)
    if where != "v":
        lay = psa.make_layout(1024, 64, 64, 64, 4)
        with pytest.raises(psa.ValidationError):
            psa.importance_sampled(q, k, lay, psa.SamplerConfig(8, 8, 0))
    # check_finite=False: no check (the caller vouches for the data)
    psa.psa_attention(q, k, v, check_finite=False, **KW)

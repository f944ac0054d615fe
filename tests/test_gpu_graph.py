"""GPU: the CUDA-graph replay of the fused forward (graph.CapturedForward) is bit-identical to the
eager call, on the capture inputs and after new inputs are copied in, for the sampled and the
antidiagonal (causal, GQA, similarity cap) estimators and for a query-block work unit."""

import pytest
import torch

from helpers import gaussian_qkv, to_dev

pytestmark = pytest.mark.gpu

CASES = {
    "cfg1_sampled_d64": dict(n=4096, d=64, b_q=64, b_k=64, levels=4, estimator="sampled-max",
                             s_q=8, s_k=8, seed=0, mask="threshold",
                             thresholds=[0.164713, 0.282366, 0.376488, 0.95], tile_len=128,
                             hq=2, hkv=2),
    "antidiag_causal_gqa": dict(n=4096, d=128, b_q=128, b_k=64, levels=4, estimator="antidiagonal",
                                stride=8, mask="threshold", thresholds=[0.16, 0.28, 0.37, 0.95],
                                sim_thresholds=[0.75, 0.7, 0.7], causal=True, tile_len=128, hq=4,
                                hkv=2),
}


def _inputs(case, seed):
    c = CASES[case]
    q, k, v = gaussian_qkv(seed, c["hq"], c["n"], c["d"], c["hkv"])
    return tuple(to_dev(x)[None].contiguous() for x in (q, k, v))


def _same(a, b):
    assert torch.equal(a.out, b.out)
    assert torch.equal(a.lse, b.lse)
    assert torch.equal(a.plan.level_map, b.plan.level_map)
    assert torch.equal(a.plan.info, b.plan.info)
    assert torch.equal(a.plan.level_counts, b.plan.level_counts)
    assert int(a.skipped.item()) == int(b.skipped.item())


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("qblocks", [None, [5, 0, 17]])
def test_graph_replay_matches_eager(case, qblocks):
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.graph import CapturedForward
    from paper_2512_04025_b200.pipeline import psa_forward_4d
    c = dict(CASES[case])
    c.pop("hq"), c.pop("hkv")
    cfg = psa.RunConfig.from_dict(c)
    q4, k4, v4 = _inputs(case, 11)
    cap = CapturedForward(q4, k4, v4, cfg, qblocks=qblocks)
    res = cap()
    torch.cuda.synchronize()
    _same(res, psa_forward_4d(q4, k4, v4, cfg, qblocks=qblocks))
    q2, k2, v2 = _inputs(case, 12)  # new inputs through the static buffers
    res = cap(q2, k2, v2)
    torch.cuda.synchronize()
    _same(res, psa_forward_4d(q2, k2, v2, cfg, qblocks=qblocks))


def test_graph_rejects_other_shapes():
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.errors import ValidationError
    from paper_2512_04025_b200.graph import CapturedForward
    c = dict(CASES["cfg1_sampled_d64"])
    c.pop("hq"), c.pop("hkv")
    q4, k4, v4 = _inputs("cfg1_sampled_d64", 3)
    cap = CapturedForward(q4, k4, v4, psa.RunConfig.from_dict(c))
    with pytest.raises(ValidationError):
        cap(q4[:, :1].contiguous())

"""GPU: determinism (the reference is "identical regardless of degree of
parallelism"). Two runs of the fused forward give bit-identical scores, level maps,
plans, O and lse; splitting the heads over several calls (what ranks do) gives the same per-head
results as one call; the backward (no atomics: per-level slabs summed in a fixed order) gives
bit-identical gradients on repeated runs."""

import pytest
import torch

from helpers import gaussian_qkv, to_dev

pytestmark = pytest.mark.gpu

CASES = {
    "sampled": dict(n=7680, d=128, b_q=120, b_k=120, levels=4, estimator="sampled-max", s_q=8,
                    s_k=8, seed=3, mask="threshold", thresholds=[0.16, 0.28, 0.37, 0.95],
                    tile_len=128, hq=4, hkv=4),
    "antidiag_causal_gqa": dict(n=8192, d=128, b_q=128, b_k=64, levels=4, estimator="antidiagonal",
                                stride=8, mask="threshold", thresholds=[0.07, 0.12, 0.16, 0.4],
                                sim_thresholds=[0.75, 0.7, 0.7], causal=True, tile_len=128, hq=8,
                                hkv=2),
}


def _setup(case, seed=21):
    import paper_2512_04025_b200 as psa
    c = dict(CASES[case])
    hq, hkv = c.pop("hq"), c.pop("hkv")
    cfg = psa.RunConfig.from_dict(c)
    q, k, v = gaussian_qkv(seed, hq, c["n"], c["d"], hkv)
    return cfg, hq, hkv, tuple(to_dev(x)[None].contiguous() for x in (q, k, v))


@pytest.mark.parametrize("case", sorted(CASES))
def test_repeated_forward_is_bit_identical(case):
    from paper_2512_04025_b200.pipeline import psa_forward_4d
    cfg, _, _, (q4, k4, v4) = _setup(case)
    a = psa_forward_4d(q4, k4, v4, cfg, keep_scores=True)
    b = psa_forward_4d(q4, k4, v4, cfg, keep_scores=True)
    assert torch.equal(a.scores, b.scores)
    assert torch.equal(a.plan.level_map, b.plan.level_map)
    assert torch.equal(a.plan.info, b.plan.info)
    # the plan rows hold info[:, 0] entries each; the rest of a row is unused workspace
    live = torch.arange(a.plan.csr.shape[1], device=a.plan.csr.device)[None] < a.plan.info[:, :1]
    assert torch.equal(a.plan.csr[live], b.plan.csr[live])
    assert torch.equal(a.out, b.out) and torch.equal(a.lse, b.lse)


@pytest.mark.parametrize("case", sorted(CASES))
def test_head_split_matches_single_call(case):
    """Per-head results do not depend on how many heads share a call (the rank-level split)."""
    from paper_2512_04025_b200.pipeline import psa_forward_4d
    cfg, hq, hkv, (q4, k4, v4) = _setup(case)
    full = psa_forward_4d(q4, k4, v4, cfg, keep_scores=True)
    g = hq // hkv
    for kv in range(hkv):  # one call per KV head with its query heads
        qs = q4[:, kv * g:(kv + 1) * g].contiguous()
        part = psa_forward_4d(qs, k4[:, kv:kv + 1].contiguous(), v4[:, kv:kv + 1].contiguous(), cfg,
                              keep_scores=True)
        sl = slice(kv * g, (kv + 1) * g)
        assert torch.equal(part.scores, full.scores[:, sl])
        assert torch.equal(part.plan.level_map, full.plan.level_map[:, sl])
        assert torch.equal(part.out, full.out[:, sl])
        assert torch.equal(part.lse, full.lse[:, sl])


def test_backward_is_bit_identical():
    import paper_2512_04025_b200 as psa
    cfg, _, _, (q4, k4, v4) = _setup("sampled")
    grads = []
    for _ in range(2):
        q, k, v = (x.clone().requires_grad_(True) for x in (q4, k4, v4))
        out, _ = psa.psa_attention_differentiable(q, k, v, cfg)
        (out.float() * torch.linspace(-1, 1, out.shape[-1], device=out.device)).sum().backward()
        grads.append((q.grad.clone(), k.grad.clone(), v.grad.clone()))
    for a, b in zip(*grads):
        assert torch.equal(a, b)

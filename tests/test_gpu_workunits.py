"""GPU: query-block work units. A call restricted to a query-block subset returns,
for every listed block, exactly the rows of the full-head call (importance rows, level map, plan,
O, lse bit-identical), for the sampled and the antidiagonal estimators, causal and GQA; and the
multi-rank partition (2 gloo ranks sharing one GPU) reassembles the single-process output
bit-for-bit (the §8e correctness criterion)."""

import os
import socket

import numpy as np
import pytest
import torch

from helpers import gaussian_qkv, to_dev

pytestmark = pytest.mark.gpu

CASES = {
    "sampled": dict(n=3840, d=128, b_q=120, b_k=120, levels=4, estimator="sampled-max", s_q=8,
                    s_k=8, seed=0, mask="threshold", thresholds=[0.16, 0.28, 0.37, 0.95],
                    tile_len=128, hq=3, hkv=3),
    "antidiag_causal_gqa": dict(n=4096, d=128, b_q=128, b_k=64, levels=4, estimator="antidiagonal",
                                stride=8, mask="threshold", thresholds=[0.16, 0.28, 0.37, 0.95],
                                sim_thresholds=[0.75, 0.7, 0.7], causal=True, tile_len=128, hq=4,
                                hkv=2),
}


def _cfg(case):
    import paper_2512_04025_b200 as psa
    c = dict(CASES[case])
    c.pop("hq"), c.pop("hkv")
    return psa.RunConfig.from_dict(c)


@pytest.mark.parametrize("case", sorted(CASES))
def test_query_block_subset_matches_full_rows(case):
    from paper_2512_04025_b200.pipeline import psa_forward_4d
    c = CASES[case]
    cfg = _cfg(case)
    q, k, v = gaussian_qkv(91, c["hq"], c["n"], c["d"], c["hkv"])
    q4, k4, v4 = (to_dev(x)[None] for x in (q, k, v))
    full = psa_forward_4d(q4, k4, v4, cfg, keep_scores=True)
    n_q = c["n"] // c["b_q"]
    rng = np.random.default_rng(5)
    for blocks in ([0], [n_q - 1, 3, 1], sorted(rng.choice(n_q, n_q // 3, replace=False).tolist())):
        sub = psa_forward_4d(q4, k4, v4, cfg, keep_scores=True, qblocks=blocks)
        bi = torch.tensor(blocks, device="cuda")
        assert torch.equal(sub.scores, full.scores[:, :, bi])
        assert torch.equal(sub.plan.level_map, full.plan.level_map[:, :, bi])
        rows = (bi[:, None] * c["b_q"] + torch.arange(c["b_q"], device="cuda")[None]).reshape(-1)
        assert torch.equal(sub.out, full.out[:, :, rows])
        assert torch.equal(sub.lse, full.lse[:, :, rows])
        units = (torch.arange(c["hq"], device="cuda")[:, None] * n_q + bi[None]).reshape(-1)
        assert torch.equal(sub.plan.info, full.plan.info[units])
        for u_sub, u_full in enumerate(units.tolist()):
            ne = int(full.plan.info[u_full, 0])
            assert torch.equal(sub.plan.csr[u_sub, :ne], full.plan.csr[u_full, :ne])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, case, q, k, v, queue):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_04025_b200.parallel import gather_partitioned, partition
        from paper_2512_04025_b200.pipeline import psa_forward_4d
        c = CASES[case]
        cfg = _cfg(case)
        n_q = c["n"] // c["b_q"]
        outs, lses = [], []
        for q_lo, q_hi, kv_lo, kv_hi, blocks in partition(c["hq"], c["hkv"], n_q, world, rank,
                                                          cfg.causal):
            q4 = q[:, q_lo:q_hi].cuda().contiguous()
            k4 = k[:, kv_lo:kv_hi].cuda().contiguous()
            v4 = v[:, kv_lo:kv_hi].cuda().contiguous()
            res = psa_forward_4d(q4, k4, v4, cfg, qblocks=blocks)
            outs.append(res.out.cpu())
            lses.append(res.lse.cpu())
        o = gather_partitioned(outs, c["hq"], c["hkv"], n_q, c["b_q"], cfg.causal)
        l_ = gather_partitioned(lses, c["hq"], c["hkv"], n_q, c["b_q"], cfg.causal)
        if rank == 0:
            queue.put((o.view(torch.int16).numpy(), l_.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_two_rank_partition_reassembles_single_gpu_output(case):
    import torch.multiprocessing as mp
    from paper_2512_04025_b200.pipeline import psa_forward_4d
    c = CASES[case]
    q, k, v = gaussian_qkv(93, c["hq"], c["n"], c["d"], c["hkv"])
    q4, k4, v4 = (torch.from_numpy(x).to(torch.bfloat16)[None] for x in (q, k, v))
    full = psa_forward_4d(q4.cuda(), k4.cuda(), v4.cuda(), _cfg(case))
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, case, q4, k4, v4, queue))
             for r in range(2)]
    for p_ in procs:
        p_.start()
    o, l_ = queue.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    assert np.array_equal(o, full.out.cpu().view(torch.int16).numpy())
    assert np.array_equal(l_, full.lse.cpu().numpy())

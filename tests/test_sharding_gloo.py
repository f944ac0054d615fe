"""CPU, world_size 2 (gloo): the (batch, head) sharding covers every head exactly once and the
optional output gather reassembles the single-process result bit-for-bit."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_04025_b200.parallel import gather_outputs, shard_heads


@pytest.mark.parametrize("hq,hkv,world", [(40, 40, 8), (12, 12, 8), (28, 4, 8), (28, 4, 3),
                                          (2, 2, 2), (40, 40, 1), (6, 3, 4), (28, 4, 5)])
def test_shards_partition_heads(hq, hkv, world):
    """Every query head on exactly one rank, ranks balanced to within one head, each rank reads
    the KV heads of its query heads, and its segments are uniform-GQA calls covering its range."""
    from paper_2512_04025_b200.parallel import shard_segments
    group = hq // hkv
    seen_q, seen_kv, sizes = [], set(), []
    for r in range(world):
        q, kv = shard_heads(hq, hkv, world, r)
        seen_q += q
        seen_kv |= set(kv)
        sizes.append(len(q))
        assert all(h // group in kv for h in q)
        covered = []
        for q_lo, q_hi, kv_lo, kv_hi in shard_segments(hq, hkv, world, r):
            g = (q_hi - q_lo) // (kv_hi - kv_lo)
            assert g * (kv_hi - kv_lo) == q_hi - q_lo
            assert all(h // group == kv_lo + (h - q_lo) // g for h in range(q_lo, q_hi))
            covered += list(range(q_lo, q_hi))
        assert covered == q
    assert sorted(seen_q) == list(range(hq)) and seen_kv == set(range(hkv))
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, hq, hkv, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(2 * hq * 8 * 4, dtype=torch.float32).reshape(2, hq, 8, 4)
        heads, _ = shard_heads(hq, hkv, world, rank)
        local = full[:, heads] * 1.0  # the "computation" of this rank's shard
        got = gather_outputs(local, hq, hkv, dst=0)
        if rank == 0:
            q.put(bool(torch.equal(got, full)))
        else:
            q.put(got is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("hq,hkv", [(6, 3), (5, 5)])
def test_gather_world2_gloo(hq, hkv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, hq, hkv, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = [q.get(timeout=5) for _ in range(2)]
    assert all(res) and all(p.exitcode == 0 for p in procs)


def _part_worker(rank, world, port, hq, hkv, n_q, b_q, causal, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_04025_b200.parallel import gather_partitioned, partition
        full = torch.arange(2 * hq * n_q * b_q * 3, dtype=torch.float32).reshape(2, hq, n_q * b_q, 3)
        pieces = []
        for q_lo, q_hi, _, _, blocks in partition(hq, hkv, n_q, world, rank, causal):
            x = full[:, q_lo:q_hi].reshape(2, q_hi - q_lo, n_q, b_q, 3)
            if blocks is not None:
                x = x[:, :, blocks]
            pieces.append(x.reshape(2, q_hi - q_lo, -1, 3) * 1.0)
        got = gather_partitioned(pieces, hq, hkv, n_q, b_q, causal, dst=0)
        q.put(bool(torch.equal(got, full)) if rank == 0 else got is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("hq,hkv,n_q,causal,world", [(3, 3, 10, False, 2), (4, 2, 9, True, 3),
                                                     (12, 12, 17, False, 8)])
def test_gather_partitioned_gloo(hq, hkv, n_q, causal, world):
    """(batch, head, query-block set) pieces of every rank reassemble the full output on rank 0."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_part_worker, args=(r, world, port, hq, hkv, n_q, 4, causal, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    res = [q.get(timeout=5) for _ in range(world)]
    assert all(res) and all(p.exitcode == 0 for p in procs)

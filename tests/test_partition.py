"""CPU: the (batch, head, query-block set) work units of parallel.partition cover
every (head, query block) exactly once, calls have uniform GQA, and the estimated per-rank cost
is balanced (max/min <= 1.05 at 8 ranks for cfg2 and cfg4)."""

import pytest

from paper_2512_04025_b200.parallel import (block_cost, head_parts, part_blocks, partition,
                                            rank_cost)


def _check_cover(hq, hkv, n_q, world, causal):
    group = hq // hkv
    seen = {}
    for r in range(world):
        for q_lo, q_hi, kv_lo, kv_hi, blocks in partition(hq, hkv, n_q, world, r, causal):
            g = (q_hi - q_lo) // (kv_hi - kv_lo)
            assert g * (kv_hi - kv_lo) == q_hi - q_lo
            assert all(h // group == kv_lo + (h - q_lo) // g for h in range(q_lo, q_hi))
            blk = range(n_q) if blocks is None else blocks
            if blocks is not None:
                assert q_hi - q_lo == 1 and list(blocks) == sorted(set(blocks))
            for h in range(q_lo, q_hi):
                for i in blk:
                    assert (h, i) not in seen, (h, i)
                    seen[(h, i)] = r
    assert len(seen) == hq * n_q


@pytest.mark.parametrize("hq,hkv,n_q,world,causal", [
    (12, 12, 273, 8, False), (28, 4, 256, 8, True), (40, 40, 630, 8, False), (2, 2, 64, 2, False),
    (12, 12, 273, 3, False), (28, 4, 256, 5, True), (28, 4, 256, 3, False), (40, 40, 630, 1, False),
    (6, 3, 10, 4, True), (1, 1, 7, 2, True)])
def test_partition_covers_every_unit_once(hq, hkv, n_q, world, causal):
    _check_cover(hq, hkv, n_q, world, causal)


@pytest.mark.parametrize("hq,hkv,n_q,causal", [(12, 12, 273, False), (28, 4, 256, True),
                                               (40, 40, 630, False), (12, 12, 273, True)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_balanced(hq, hkv, n_q, causal, world):
    costs = [rank_cost(partition(hq, hkv, n_q, world, r, causal), n_q, causal)
             for r in range(world)]
    assert max(costs) / min(costs) <= 1.05, costs


def test_zigzag_parts_equal_cost():
    n_q = 256
    for parts in (2, 4, 8):
        costs = [block_cost(part_blocks(n_q, parts, p, True), n_q, True) for p in range(parts)]
        assert max(costs) / min(costs) <= 1.02
    assert head_parts(12, 8) == 2 and head_parts(28, 8) == 2 and head_parts(40, 8) == 1

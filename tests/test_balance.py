"""balance.py drop-in (reference balance.py:45-73) and the per-block sharding report."""
import random

import pytest

from paper_2602_02016_b200 import balance


def test_greedy_balance_known_answer():
    a = balance.greedy_balance([(0, 5), (1, 9), (2, 5), (3, 1), (4, 9)], 2)
    # sorted: (1,9), (4,9), (0,5), (2,5), (3,1); ties on load -> lowest worker
    assert [w.layer_ids for w in a.workers] == [[1, 0, 3], [4, 2]]
    assert [w.load for w in a.workers] == [15, 14]
    rep = balance.simulate_sync_cost(a, balance.CostModel(compute_per_param=2.0, broadcast_per_param=0.5))
    assert rep.makespan == 30.0 and rep.broadcast_volume == 14.5 and rep.worker_loads == (15, 14)


@pytest.mark.parametrize("bad,msg", [(([], 2), "no layers"), (([(0, 1)], 0), "at least one worker"),
                                     (([(0, 0)], 1), "non-positive"), (([(0, 1), (0, 2)], 1), "duplicate")])
def test_greedy_balance_validation(bad, msg):
    with pytest.raises(ValueError, match=msg):
        balance.greedy_balance(*bad)


def test_matches_reference_balancer(reference):
    import blockshampoo.balance as ref

    rng = random.Random(5)
    for _ in range(50):
        n, w = rng.randint(1, 40), rng.randint(1, 9)
        sizes = [(i, rng.choice([1, 2, 3, 5, 8, 13, 1000])) for i in rng.sample(range(100), n)]
        a, b = balance.greedy_balance(sizes, w), ref.greedy_balance(sizes, w)
        assert [x.layer_ids for x in a.workers] == [x.layer_ids for x in b.workers]
        assert [x.load for x in a.workers] == [x.load for x in b.workers]
        ra, rb = balance.simulate_sync_cost(a), ref.simulate_sync_cost(b)
        assert (ra.makespan, ra.broadcast_volume, ra.worker_loads) == (rb.makespan, rb.broadcast_volume,
                                                                       rb.worker_loads)


def test_block_report_953m():
    from paper_2602_02016_b200.sharded import units_of
    from paper_2602_02016_b200.shampoo import build_layout
    from tests.golden.cases import llama_953m

    layers, _ = build_layout(llama_953m(), 1024)
    units = units_of(layers)
    for w in (2, 4, 8):
        rep = balance.block_report(units, balance.block_balance(units, w))
        assert sum(rep.units_per_rank) == len(units)
        assert rep.imbalance < 1.02  # LPT over 960+ near-equal blocks
        assert rep.allgather_bytes > 0

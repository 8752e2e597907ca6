"""The fused route + exchange's placement (hm_dist_exchange_plan; DESIGN.md §9
NEXT-2), on CPU: every rank stores its run for owner r at off[r] in r's
window, so over all ranks each owner's first recv positions are written
exactly once, by the pairs it owns, and the window size cap is the largest
receive count.  Simulated for 2, 3 and 5 ranks on the generator's keys with
the oracle's level-1 function (owner(b) = floor(b G / n))."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2508_11443_b200 import hm
from workloads import gen


@pytest.mark.parametrize("world,n,seed", [(2, 5000, 0), (3, 4001, 2), (5, 20_000, 7), (1, 100, 0)])
def test_exchange_plan_places_every_pair_once(world, n, seed):
    keys = gen.u64_keys(n)
    owner = (O.level1_buckets(keys, n, seed, 0).astype(np.int64) * world) // n
    ranks = np.minimum(np.arange(n) * world // n, world - 1)  # the input split over the ranks
    Cm = np.zeros((world, world), np.uint64)
    for q in range(world):
        Cm[q] = np.bincount(owner[ranks == q], minlength=world)
    plans = [hm.dist_exchange_plan(Cm, world, q) for q in range(world)]
    caps = {p[1] for p in plans}
    assert len(caps) == 1  # the same symmetric window size on every rank
    cap = caps.pop()
    recv = [p[2] for p in plans]
    assert recv == [int(Cm[:, r].sum()) for r in range(world)] and cap == max(recv)
    # every rank writes its run for owner r at off[r] .. off[r] + C[q][r]
    win = [np.full(cap, -1, np.int64) for _ in range(world)]
    for q in range(world):
        off = plans[q][0]
        mine = np.nonzero(ranks == q)[0]
        for r in range(world):
            run = mine[owner[mine] == r]
            seg = win[r][off[r]:off[r] + len(run)]
            assert (seg == -1).all()  # (no overlap with another sender's run)
            win[r][off[r]:off[r] + len(run)] = run
    for r in range(world):
        got = win[r][:recv[r]]
        assert (got >= 0).all() and (win[r][recv[r]:] == -1).all()
        assert np.array_equal(np.sort(got), np.nonzero(owner == r)[0])
    with pytest.raises(hm.HMError):
        hm.dist_exchange_plan(Cm, world, world)

"""Pins of the oracle's expert migration (NEXT-2; §VI, Alg. 2):
hand-worked instances, an independent brute-force replay of every iteration, invariants,
and the paper's migration-cost table."""
import itertools
import math
import os

import numpy as np
import pytest

import synth
from oracle import migration as mig
from oracle import moe_ref as ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_worked_instances():
    # [[8,6],[1,1]]: s=[14,2], delta=12; swaps (8,1) and (6,1) both give delta'=2 (gain 10):
    # the first in (i,j) order wins -> [[1,6],[8,1]] (s=[7,9]); then no swap reduces 2 -> c=1
    G, c, swaps = mig.hill_climb([[8, 6], [1, 1]])
    assert G == [[1, 6], [8, 1]] and c == 1 and swaps == [(0, 0, 1, 0)]
    # [[10,1],[2,3]]: s=[11,5], delta=6; every swap gives delta' >= 8 -> no move
    G, c, _ = mig.hill_climb([[10, 1], [2, 3]])
    assert G == [[10, 1], [2, 3]] and c == 0
    # balanced input: nothing to do
    assert mig.hill_climb([[3, 3], [3, 3], [3, 3]])[1] == 0
    # three groups, worked by hand: s=[11,10,2] -> swap (9,1) [tie with (2,1), first wins]
    # -> [[1,2],[5,5],[9,1]] s=[3,10,10]; k+=1 (first max), k-=0: swap (5,1) -> s=[7,6,10];
    # k+=2, k-=1, delta=4: no swap reduces it -> stop, c=2
    G, c, swaps = mig.hill_climb([[9, 2], [5, 5], [1, 1]])
    assert G == [[5, 2], [1, 5], [9, 1]] and c == 2
    assert swaps == [(0, 0, 2, 0), (1, 0, 0, 0)]
    # Alg. 2 only ever swaps between the max and the min group: [[9,1],[5,5],[1,1]] has
    # s=[10,10,2] and no max/min swap reduces delta=8, so it stops at once (a local optimum)
    assert mig.hill_climb([[9, 1], [5, 5], [1, 1]])[1] == 0


def brute_replay(groups, swaps, T=100):
    """Re-derive every iteration independently: enumerate all (i, j) with itertools, pick the
    largest strict reduction of |s+ - s-| (first in order on ties) and compare."""
    G = [list(g) for g in groups]
    for t in range(T):
        s = [sum(g) for g in G]
        kp = min(range(len(G)), key=lambda k: (-s[k], k))
        km = min(range(len(G)), key=lambda k: (s[k], k))
        delta = s[kp] - s[km]
        cands = []
        for i, j in itertools.product(range(len(G[kp])), range(len(G[km]))):
            d2 = abs((s[kp] - G[kp][i] + G[km][j]) - (s[km] - G[km][j] + G[kp][i]))
            if d2 < delta:
                cands.append((delta - d2, -i, -j))
        if not cands:
            assert t == len(swaps)
            return G
        gain, ni, nj = max(cands)
        assert swaps[t] == (kp, -ni, km, -nj), (t, swaps[t], (kp, -ni, km, -nj))
        G[kp][-ni], G[km][-nj] = G[km][-nj], G[kp][-ni]
    assert len(swaps) == T
    return G


@pytest.mark.parametrize("seed", range(12))
def test_hill_climb_matches_brute_force_replay_and_invariants(seed):
    rng = np.random.default_rng(seed)
    K, n = int(rng.integers(2, 9)), int(rng.integers(1, 9))
    groups = [list(map(int, rng.integers(0, 1000, n))) for _ in range(K)]
    G, c, swaps = mig.hill_climb(groups)
    assert c == len(swaps) <= 100
    assert brute_replay(groups, swaps) == G
    assert sorted(sum(G, [])) == sorted(sum(groups, []))        # items preserved
    assert all(len(g) == n for g in G)                           # group sizes preserved
    # every applied swap strictly reduced the difference of the two groups it touched
    H = [list(g) for g in groups]
    for kp, i, km, j in swaps:
        before = abs(sum(H[kp]) - sum(H[km]))
        H[kp][i], H[km][j] = H[km][j], H[kp][i]
        assert abs(sum(H[kp]) - sum(H[km])) < before


def test_rebalance_placement_zipf_config():
    """V3-like Zipf routing (reading R11): the migration brings the hottest rank close to the
    mean; the result is a permutation, unmoved experts keep their slots."""
    cfg = synth.CONFIGS["dsv3"]
    ep = 8
    T = 4096
    L = synth.random_logits(T, cfg.E, seed=1).numpy() + synth.zipf_bias(cfg).numpy()[None, :]
    idx, _ = ref.route(L, cfg.k)
    loads = np.bincount(idx.ravel(), minlength=cfg.E)
    before = mig.rank_loads(loads, np.arange(cfg.E), ep)
    place, c = mig.rebalance_placement(loads, ep)
    after = mig.rank_loads(loads, place, ep)
    assert sorted(place) == list(range(cfg.E)) and c > 0
    assert after.sum() == before.sum() == T * cfg.k
    assert after.max() < before.max() and after.max() / after.mean() < 1.05 < before.max() / before.mean()
    moved = np.nonzero(place != np.arange(cfg.E))[0]
    assert len(moved) <= 2 * c
    # recv layout under a placement: each owner's segments hold exactly its experts' rows
    plan = ref.dispatch_plan(idx, cfg.E, 1, None, align=128, placement=np.arange(cfg.E))
    assert plan["layouts"][0]["expert_rows"].sum() == T * cfg.k


def test_migration_cost_table_golden():
    """a complete reassignment moves 48 E d f / G bytes per GPU."""
    for line in open(os.path.join(GOLDEN, "migration_worst_case.txt")):
        if line.startswith("#") or not line.strip():
            continue
        model, E, d, f, gb, ms, unit = line.split()
        E, d, f = int(E), int(d), int(f)
        b = mig.migration_bytes(E // 8, d, f)
        if unit == "GiB":
            assert math.ceil(b / 2**30 * 100 - 1e-9) / 100 == float(gb), model


def test_imbalance_trigger_hand_worked():
    """Reading R20: imbalance = max_q s_q / mean_q s_q.  E=4 on EP=2, contiguous placement:
    loads [6, 2, 1, 1] -> s = [8, 2], mean 5 -> 1.6; after swapping experts 1 and 2 the ranks
    hold [6, 1] and [2, 1] -> s = [7, 3] -> 1.4; a perfectly balanced load is exactly 1."""
    assert mig.imbalance([6, 2, 1, 1], [0, 1, 2, 3], 2) == 1.6
    assert mig.imbalance([6, 2, 1, 1], [0, 2, 1, 3], 2) == 1.4
    assert mig.imbalance([3, 3, 3, 3], [0, 1, 2, 3], 4) == 1.0
    assert mig.imbalance([0, 0, 0, 0], [0, 1, 2, 3], 2) == 1.0
    assert mig.should_migrate([6, 2, 1, 1], [0, 1, 2, 3], 2, 1.5)
    assert not mig.should_migrate([6, 2, 1, 1], [0, 1, 2, 3], 2, 1.6)   # strictly above
    # Alg. 2 never raises the imbalance it is triggered on (it only applies improving swaps)
    rng = np.random.default_rng(3)
    for _ in range(50):
        loads = rng.integers(0, 1000, 16)
        new, _ = mig.rebalance_placement(loads, 4)
        assert mig.imbalance(loads, new, 4) <= mig.imbalance(loads, np.arange(16), 4)

"""Expert migration (§VI).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* `hill_climb` is Alg. 2 "Hill-Climbing Swap-Based Minimal Rebalancing"
  written out step by step in the paper's notation: groups G_1..G_K of item loads (here:
  EP ranks holding E/EP experts each, loads = routed token counts), at most T = 100
  iterations, each applying the single swap between the most- and least-loaded groups that
  reduces their difference the most.
  Readings (R16): argmax / argmin ties go to the lowest group index; candidate
  pairs are visited in (i, j) index order and the strict ">" keeps the first best one; the
  swapped items keep their slot positions (slot i of G_k+ <-> slot j of G_k-).
* `placement_from_groups` turns the groups into the expert -> (owner, slot) map the layer uses.
* `imbalance` / `should_migrate` are the external scheduler's trigger (it
  "inspects the growing load imbalance, and whenever it crosses a pre-determined threshold"
  runs Alg. 2).  Reading R20: imbalance = max_q s_q / mean_q s_q over the EP
  ranks' routed rows s_q under the current placement (1 = balanced; the step time of an EP
  layer follows its most-loaded rank), migrate iff imbalance > threshold.
* `migration_bytes` is the paper's cost: 48 d f bytes per moved expert.
"""
from __future__ import annotations

import numpy as np


def hill_climb(groups, T=100):
    """groups: list of K lists of item loads (the lists are copied).  Returns
    (groups after rebalancing, swap count c, list of swaps (k_plus, i, k_minus, j))."""
    G = [list(g) for g in groups]
    c = 0
    swaps = []
    for _t in range(T):
        s = [sum(g) for g in G]
        k_plus = int(np.argmax(s))          # first maximum
        k_minus = int(np.argmin(s))         # first minimum
        delta = s[k_plus] - s[k_minus]
        best_swap = None
        best_gain = 0
        for i, n1 in enumerate(G[k_plus]):
            for j, n2 in enumerate(G[k_minus]):
                d2 = abs((s[k_plus] - n1 + n2) - (s[k_minus] - n2 + n1))
                if d2 < delta and (delta - d2) > best_gain:
                    best_gain = delta - d2
                    best_swap = (i, j)
        if best_swap is None:
            break
        i, j = best_swap
        G[k_plus][i], G[k_minus][j] = G[k_minus][j], G[k_plus][i]
        c += 1
        swaps.append((k_plus, i, k_minus, j))
    return G, c, swaps


def rebalance_placement(loads, ep, placement=None, T=100):
    """loads[e] = token rows routed to expert e.  placement[e] = global slot of expert e
    (owner = slot // E_l, local slot = slot % E_l); default contiguous (slot = e).
    Runs Alg. 2 on the groups {loads of the experts in owner q's slots} and returns the new
    placement (same slot positions for experts that did not move) and the swap count."""
    loads = np.asarray(loads, np.int64)
    E = loads.size
    E_l = E // ep
    placement = np.arange(E) if placement is None else np.asarray(placement, np.int64)
    expert_at = np.empty(E, np.int64)
    expert_at[placement] = np.arange(E)
    groups = [[int(loads[expert_at[q * E_l + el]]) for el in range(E_l)] for q in range(ep)]
    ids = [[int(expert_at[q * E_l + el]) for el in range(E_l)] for q in range(ep)]
    _, c, swaps = hill_climb(groups, T)
    for kp, i, km, j in swaps:                      # replay the swaps on the expert ids
        ids[kp][i], ids[km][j] = ids[km][j], ids[kp][i]
    new_place = np.empty(E, np.int64)
    for q in range(ep):
        for el in range(E_l):
            new_place[ids[q][el]] = q * E_l + el
    return new_place, c


def rank_loads(loads, placement, ep):
    """Rows received per owner rank under a placement."""
    loads = np.asarray(loads, np.int64)
    E = loads.size
    out = np.zeros(ep, np.int64)
    np.add.at(out, np.asarray(placement) // (E // ep), loads)
    return out


def imbalance(loads, placement, ep):
    """max over ranks / mean over ranks of the routed rows (reading R20); 1.0 for no load."""
    s = rank_loads(loads, placement, ep)
    tot = int(s.sum())
    return 1.0 if tot == 0 else float(s.max()) * ep / tot


def should_migrate(loads, placement, ep, threshold):
    return imbalance(loads, placement, ep) > threshold


def migration_bytes(n_experts_moved, d, f, bytes_per_param=16):
    """each migrated expert moves 3 d f parameters at 16 B/param = 48 d f bytes."""
    return bytes_per_param * 3 * d * f * n_experts_moved

"""Pins of the deduplicated all-to-all oracle (oracle/dedup.py, SURVEY.md §8(f) NEXT-4,
DESIGN.md reading R18) against brute force, closed forms on the balanced fixture, special
cases that reduce to the plain dispatch, and the plain layer's own result."""
import numpy as np
import pytest

import synth
from oracle import dedup as dd
from oracle import moe_ref as ref


def brute_pairs(dest_row, idx, placement, E_l, ep):
    """Pure-Python loops: walk tokens in order, one pair per distinct owner of a kept slot."""
    T_r, k = idx.shape
    tslot = [[-1] * ep for _ in range(T_r)]
    n = [0] * ep
    for t in range(T_r):
        owners = set()
        for j in range(k):
            if dest_row[t][j] >= 0:
                owners.add(int(placement[int(idx[t][j])]) // E_l)
        for q in sorted(owners):
            tslot[t][q] = n[q]
            n[q] += 1
    return np.array(tslot), np.array(n)


def random_plan(T_r, E, k, ep, cf, seed, placement=None):
    L = synth.random_logits(ep * T_r, E, seed=seed).numpy()
    idx, gates = ref.route(L, k)
    C = ref.capacity(cf, k, T_r, E)
    return idx, gates, dd.plan(idx, gates, E, ep, C, align=128, placement=placement)


@pytest.mark.parametrize("E,k,ep,cf", [(8, 2, 2, 1.25), (16, 4, 4, 0.5), (64, 6, 4, 1.25),
                                       (32, 8, 8, 0.0), (8, 2, 1, 1.0)])
def test_pairs_match_brute_force(E, k, ep, cf):
    T_r = 96
    idx, _, P = random_plan(T_r, E, k, ep, cf, seed=E + k + ep)
    place = np.arange(E)
    for r in range(ep):
        pr = P["pairs"][r]
        tslot, n = brute_pairs(P["base"]["ranks"][r]["dest_row"], idx[r * T_r:(r + 1) * T_r],
                               place, E // ep, ep)
        np.testing.assert_array_equal(pr["tslot"], tslot)
        np.testing.assert_array_equal(pr["ntok"], n)


def test_pairs_under_a_migrated_placement():
    E, k, ep, T_r = 16, 4, 4, 64
    place = np.random.default_rng(3).permutation(E)
    idx, _, P = random_plan(T_r, E, k, ep, 1.25, seed=5, placement=place)
    for r in range(ep):
        tslot, n = brute_pairs(P["base"]["ranks"][r]["dest_row"], idx[r * T_r:(r + 1) * T_r],
                               place, E // ep, ep)
        np.testing.assert_array_equal(P["pairs"][r]["tslot"], tslot)
        np.testing.assert_array_equal(P["pairs"][r]["ntok"], n)


@pytest.mark.parametrize("E,k,ep", [(16, 2, 4), (8, 4, 4), (32, 8, 4), (64, 8, 8)])
def test_balanced_fixture_closed_form(E, k, ep):
    """l[t,e] = -((e - k t_g) mod E): token t_g takes the k consecutive experts from
    s = k t_g mod E.  When E_l | k or k | E_l, s is aligned, the window covers exactly
    max(1, k/E_l) owners, so every source sends max(1, k/E_l) * T_r pairs, split evenly:
    ntok[r][q] = max(1, k/E_l) * T_r / EP."""
    E_l = E // ep
    assert E_l % k == 0 or k % E_l == 0
    T_r = 4 * E
    L = np.concatenate([synth.balanced_logits(T_r, E, k, r).numpy() for r in range(ep)])
    idx, gates = ref.route(L, k)
    P = dd.plan(idx, gates, E, ep, None)
    per_tok = max(1, k // E_l)
    np.testing.assert_array_equal(P["ntok_all"], np.full((ep, ep), per_tok * T_r // ep))
    # the dedup egress is the plain egress divided by the slots a token keeps per owner
    plain = 2 * T_r * k * 4 * (ep - 1) // ep               # d = 4
    assert (dd.egress_bytes(P["ntok_all"], 4) * (k // per_tok) == plain).all()


@pytest.mark.parametrize("E,k,ep", [(8, 2, 8), (16, 1, 4), (4, 3, 4)])
def test_one_slot_per_owner_is_the_plain_dispatch(E, k, ep):
    """E_l = 1 (distinct experts are distinct owners) or k = 1: every pair carries exactly
    one slot, ntok[r][q] = counts[r][experts of q], and the bytes equal the plain dispatch."""
    T_r = 80
    idx, _, P = random_plan(T_r, E, k, ep, 1.25, seed=11)
    E_l = E // ep
    cm = P["base"]["counts_all"]
    np.testing.assert_array_equal(P["ntok_all"], cm.reshape(ep, ep, E_l).sum(axis=2))
    for q in range(ep):
        assert ((P["rlist"][q] >= 0).sum(axis=1) == 1).all()


@pytest.mark.parametrize("E,k,ep,cf", [(16, 4, 4, 1.0), (64, 6, 8, 1.25), (8, 2, 2, 0.0)])
def test_pair_invariants(E, k, ep, cf):
    T_r = 128
    idx, gates, P = random_plan(T_r, E, k, ep, cf, seed=21)
    E_l = E // ep
    cm = P["base"]["counts_all"]
    per_owner_rows = cm.reshape(ep, ep, E_l).sum(axis=2)          # [r][q] plain rows
    n = P["ntok_all"]
    assert (n <= per_owner_rows).all() and (n <= T_r).all()
    assert ((n > 0) == (per_owner_rows > 0)).all()
    # every kept slot is named by exactly one rlist entry, at its plain receive row
    for q in range(ep):
        rl = P["rlist"][q]
        named = np.sort(rl[rl >= 0])
        want = np.sort(P["base"]["recv_row"][P["base"]["owner"] == q])
        np.testing.assert_array_equal(named, want[want >= 0])
        u, j = np.nonzero(rl >= 0)
        t = P["tok"][q][u]
        np.testing.assert_array_equal(rl[u, j], P["base"]["recv_row"][t, j])
        np.testing.assert_array_equal(P["glist"][q][u, j], gates[t, j])
        assert (P["glist"][q][rl < 0] == 0).all()
        # token rows ordered (source, ascending t)
        key = P["src"][q] * (ep * T_r) + P["tok"][q]
        assert (np.diff(key) > 0).all()


def test_expand_rebuilds_the_plain_receive_buffer():
    """Step 3: expanding the pair rows reproduces, bit for bit, the expert-major buffer the
    plain dispatch builds (moe_ref.dispatch_plan recv_row, 128-aligned segments)."""
    E, k, ep, T_r, d = 16, 4, 4, 64, 8
    idx, gates, P = random_plan(T_r, E, k, ep, 1.25, seed=31)
    x = np.random.default_rng(0).standard_normal((ep * T_r, d))
    base = P["base"]
    for q in range(ep):
        lay = base["layouts"][q]
        n_rows = int(lay["seg_base"][-1])
        plain = np.zeros((n_rows, d))
        t, j = np.nonzero((base["owner"] == q) & (base["recv_row"] >= 0))
        plain[base["recv_row"][t, j]] = x[t]
        xt = x[P["tok"][q]]                                       # what the pairs carry
        np.testing.assert_array_equal(dd.expand(xt, P["rlist"][q], n_rows), plain)


@pytest.mark.parametrize("ep,cf", [(4, 1.25), (2, 0.5), (8, 0.0)])
def test_pair_reduction_reproduces_the_layer(ep, cf):
    """Steps 4-5 regroup sum_j into sum_q sum_{j on q}: y and the expert part of dx from the
    pair partials equal moe_ref's plain forward / backward (fp64, to rounding)."""
    E, k, T_r, d, f = 16, 4, 32, 8, 16
    T = ep * T_r
    rng = np.random.default_rng(41)
    x = rng.standard_normal((T, d))
    Wg = rng.standard_normal((E, d, f)) / np.sqrt(d)
    Wu = rng.standard_normal((E, d, f)) / np.sqrt(d)
    Wd = rng.standard_normal((E, f, d)) / np.sqrt(f)
    L = synth.random_logits(T, E, seed=43).numpy()
    fw = ref.moe_forward(x, L, Wg, Wu, Wd, k, cf, ep)
    dy = rng.standard_normal((T, d))
    bw = ref.moe_backward(fw, dy, Wg, Wu, Wd)
    P = dd.plan(fw["topk_idx"], fw["gates"], E, ep, fw["C"], align=128)
    base = P["base"]
    kept = base["recv_row"] >= 0
    # O and dX rows in each owner's receive layout, from the plain oracle
    dX_slots = np.zeros((T, k, d))
    for e in range(E):
        c = fw["cache"][e]
        if c is None:
            continue
        t, j, G, U, H = c
        dO = fw["gates"][t, j][:, None] * dy[t]
        dX_slots[t, j] = ref.expert_backward(x[t], G, U, H, dO, Wg[e], Wu[e], Wd[e])["dX"]
    y = np.zeros((T, d))
    dx = np.zeros((T, d))
    parts_y = [np.zeros((P["layout"]["pair_rows"][r], d)) for r in range(ep)]
    parts_dx = [np.zeros((P["layout"]["pair_rows"][r], d)) for r in range(ep)]
    for q in range(ep):
        n_rows = int(base["layouts"][q]["seg_base"][-1])
        O_r = np.zeros((n_rows, d))
        dX_r = np.zeros((n_rows, d))
        t, j = np.nonzero((base["owner"] == q) & kept)
        O_r[base["recv_row"][t, j]] = fw["O_slots"][t, j]
        dX_r[base["recv_row"][t, j]] = dX_slots[t, j]
        py = dd.reduce_pairs(O_r, P["rlist"][q], P["glist"][q])
        pdx = dd.reduce_pairs(dX_r, P["rlist"][q])
        for u in range(py.shape[0]):                               # owner -> source rows
            r, tt = P["src"][q][u], P["tok"][q][u] - P["src"][q][u] * T_r
            row = P["layout"]["pair_base"][r, q] + P["pairs"][r]["tslot"][tt, q]
            parts_y[r][row] = py[u]
            parts_dx[r][row] = pdx[u]
    for r in range(ep):
        sl = slice(r * T_r, (r + 1) * T_r)
        y[sl] = dd.gather_pairs(parts_y[r], P["pairs"][r], P["layout"]["pair_base"][r])
        dx[sl] = dd.gather_pairs(parts_dx[r], P["pairs"][r], P["layout"]["pair_base"][r])
    np.testing.assert_allclose(y, fw["y"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(dx, bw["dx_experts"], rtol=0, atol=1e-12)
    # dg from the owner side: <dy_t, O_{t,j}> for kept slots == the plain dgates
    dg = np.where(kept, np.einsum("td,tjd->tj", dy, fw["O_slots"]), 0.0)
    np.testing.assert_allclose(dg, bw["dgates"], rtol=0, atol=1e-12)


def test_layout_bases():
    n = np.array([[3, 0, 2], [1, 4, 0], [0, 2, 5]])
    lay = dd.layout(n)
    np.testing.assert_array_equal(lay["tok_base"], [[0, 3, 4], [0, 0, 4], [0, 2, 2]])
    np.testing.assert_array_equal(lay["pair_base"], [[0, 3, 3], [0, 1, 5], [0, 0, 2]])
    np.testing.assert_array_equal(lay["tok_rows"], [4, 6, 7])
    np.testing.assert_array_equal(lay["pair_rows"], [5, 5, 7])
    np.testing.assert_array_equal(dd.egress_bytes(n, 4), np.array([2, 1, 2]) * 8)

"""Pins of the oracle's capacity / positions / permutation / receive placement
(F2, F3) against brute force, fixtures with known answers and invariants."""
import numpy as np
import pytest

import synth
from oracle import moe_ref as ref


def brute_positions(topk, E, C):
    """Pure-Python loops: visit assignments in slot-major order a = j*T_r + t."""
    T_r, k = topk.shape
    seen = [0] * E
    p = [[0] * k for _ in range(T_r)]
    for j in range(k):
        for t in range(T_r):
            e = int(topk[t][j])
            p[t][j] = seen[e]
            seen[e] += 1
    kept = [[(C is None) or (p[t][j] < C) for j in range(k)] for t in range(T_r)]
    counts = [0] * E
    for t in range(T_r):
        for j in range(k):
            if kept[t][j]:
                counts[int(topk[t][j])] += 1
    off = [0] * E
    for e in range(1, E):
        off[e] = off[e - 1] + counts[e - 1]
    dest = [[off[int(topk[t][j])] + p[t][j] if kept[t][j] else -1 for j in range(k)]
            for t in range(T_r)]
    return np.array(p), np.array(kept), np.array(counts), np.array(dest)


@pytest.mark.parametrize("cf", [1.25, 1.0, 0.5, 0.0])
@pytest.mark.parametrize("E,k,T_r", [(8, 2, 256), (16, 4, 100), (64, 6, 96)])
def test_positions_match_brute_force(E, k, T_r, cf):
    L = synth.random_logits(T_r, E, seed=E * k + T_r).numpy()
    idx, _ = ref.route(L, k)
    C = ref.capacity(cf, k, T_r, E)
    pos = ref.positions(idx, E, C)
    p, kept, counts, dest = brute_positions(idx, E, C)
    assert (pos["p"] == p).all()
    assert (pos["kept"] == kept).all()
    assert (pos["counts"] == counts).all()
    assert (pos["dest_row"] == dest).all()


def test_capacity_values():
    # reading R4 at the configs: tiny 80; Mixtral 2560/1280/640/320; DS 240
    assert ref.capacity(1.25, 2, 256, 8) == 80
    for ep, c in [(1, 2560), (2, 1280), (4, 640), (8, 320)]:
        assert ref.capacity(1.25, 2, 8192 // ep, 8) == c
    assert ref.capacity(1.25, 6, 2048, 64) == 240
    assert ref.capacity(1.25, 8, 4096, 256) == 160
    assert ref.capacity(0.0, 8, 4096, 256) is None
    # cf is an fp32 value: 0.6f = 0.6000000238 -> 2*1500*0.6f/8 = 225.0000089 -> 226
    assert ref.capacity(0.6, 2, 1500, 8) == 226
    assert ref.capacity(0.5, 2, 1500, 8) == 188


def test_drop_priority_fixture_is_slot_major():
    """Every token picks {0,1}; expert 0 is slot 0 for odd t, slot 1 for even t.
    cf=2, E=8, k=2 -> C = T_r/2: expert 0 keeps exactly the odd tokens (its slot-0
    assignments come first), expert 1 exactly the even tokens."""
    T_r, E, k = 64, 8, 2
    L = synth.drop_priority_logits(T_r, E).numpy()
    idx, _ = ref.route(L, k)
    assert (np.sort(idx, 1) == [0, 1]).all()
    C = ref.capacity(2.0, k, T_r, E)
    assert C == T_r // 2
    pos = ref.positions(idx, E, C)
    t = np.arange(T_r)
    kept_e0 = sorted(t[((idx == 0) & pos["kept"]).any(1)])
    kept_e1 = sorted(t[((idx == 1) & pos["kept"]).any(1)])
    assert kept_e0 == list(t[t % 2 == 1])
    assert kept_e1 == list(t[t % 2 == 0])
    assert list(pos["counts"][:2]) == [C, C]


@pytest.mark.parametrize("E,k,T_r,ep", [(8, 2, 256, 1), (8, 2, 1024, 8), (64, 6, 2048, 8),
                                         (256, 8, 64, 8)])
def test_balanced_fixture_exact_counts(E, k, T_r, ep):
    for r in range(ep):
        L = synth.balanced_logits(T_r, E, k, ep_rank=r).numpy()
        idx, g = ref.route(L, k)
        pos = ref.positions(idx, E, ref.capacity(1.25, k, T_r, E))
        assert pos["kept"].all()
        assert (pos["counts"] == k * T_r // E).all()


def test_invariants_counts_drops_prefix():
    T_r, E, k = 512, 8, 2
    L = synth.random_logits(T_r, E, seed=77).numpy()
    L[:, 3] += 2.0                                 # overload expert 3 -> drops
    idx, _ = ref.route(L, k)
    C = ref.capacity(1.0, k, T_r, E)
    pos = ref.positions(idx, E, C)
    drops = (~pos["kept"]).sum()
    assert drops > 0
    assert pos["counts"].sum() + drops == T_r * k            # every slot kept or dropped
    assert (pos["counts"] <= C).all()
    assert (pos["hist"] == np.bincount(idx.ravel(), minlength=E)).all()
    # drop-prefix: a dropped (t,j) on e => every later assignment on e is dropped
    a = np.arange(T_r * k).reshape(k, T_r).T
    for e in range(E):
        m = idx == e
        dropped_a = a[m & ~pos["kept"]]
        if dropped_a.size:
            assert (~pos["kept"][m & (a > dropped_a.min())]).all()
    # dest_row is a bijection onto [0, sum counts)
    rows = pos["dest_row"][pos["kept"]]
    assert sorted(rows) == list(range(pos["counts"].sum()))
    # cf -> infinity == dropless
    big = ref.positions(idx, E, ref.capacity(1e9, k, T_r, E))
    free = ref.positions(idx, E, None)
    assert (big["dest_row"] == free["dest_row"]).all()


def test_permute_then_unpermute_identity():
    T_r, E, k, d = 128, 8, 2, 16
    x = synth.tokens(synth.CONFIGS["tiny"], T=T_r).float().numpy()[:, :d]
    idx, _ = ref.route(synth.random_logits(T_r, E, seed=4).numpy(), k)
    pos = ref.positions(idx, E, ref.capacity(1.0, k, T_r, E))
    xs = ref.permute_rows(x, pos["dest_row"], pos["counts"].sum())
    for t in range(T_r):
        for j in range(k):
            if pos["kept"][t, j]:
                assert (xs[pos["dest_row"][t, j]] == x[t]).all()
    n_kept = pos["kept"].sum(1)
    back = ref.permute_bwd(xs, pos["dest_row"])
    np.testing.assert_array_equal(back, n_kept[:, None] * x.astype(np.float64))


def brute_recv_rows(topk, E, ep, C, align):
    """Enumerate the receive buffer of every owner in (local expert, source, p) order."""
    T, k = topk.shape
    T_r, E_l = T // ep, E // ep
    pos = [ref.positions(topk[r * T_r:(r + 1) * T_r], E, C) for r in range(ep)]
    row = -np.ones((T, k), np.int64)
    for q in range(ep):
        cursor = 0
        for el in range(E_l):
            e = q * E_l + el
            start = cursor
            for r in range(ep):
                items = []
                for t in range(T_r):
                    for j in range(k):
                        if topk[r * T_r + t, j] == e and pos[r]["kept"][t, j]:
                            items.append((pos[r]["p"][t, j], t, j))
                for p, t, j in sorted(items):
                    row[r * T_r + t, j] = cursor
                    cursor += 1
            n = cursor - start
            cursor = start + (-(-n // align)) * align
    return row


@pytest.mark.parametrize("ep,align", [(1, 1), (2, 1), (4, 128), (8, 16)])
def test_recv_layout_matches_enumeration(ep, align):
    T, E, k = 256, 8, 2
    idx, _ = ref.route(synth.random_logits(T, E, seed=ep).numpy(), k)
    C = ref.capacity(1.25, k, T // ep, E)
    plan = ref.dispatch_plan(idx, E, ep, C, align=align)
    assert (plan["recv_row"] == brute_recv_rows(idx, E, ep, C, align)).all()
    for q, lay in enumerate(plan["layouts"]):
        assert (lay["recv_counts"] == plan["counts_all"][:, q * (E // ep):(q + 1) * (E // ep)].T).all()
        assert (lay["seg_base"] % align == 0).all()


def test_equal_split_dispatch_is_the_transpose_law():
    """Balanced fixture at EP=4 with one expert per rank (E_l=1, so the expert-major
    receive order coincides with source order): the dispatch moves exactly the flat
    all-to-all of the send buffers (SPEC.md:476 transpose law, SPEC.md:495-503
    brute-force N^2 copy)."""
    ep, E, k, T_r, d = 4, 4, 2, 64, 4
    T = ep * T_r
    L = np.concatenate([synth.balanced_logits(T_r, E, k, r).numpy() for r in range(ep)])
    idx, _ = ref.route(L, k)
    C = ref.capacity(1.25, k, T_r, E)
    plan = ref.dispatch_plan(idx, E, ep, C)
    # origin-encoded payload: row value = (source rank, t, j)
    send = []
    for r in range(ep):
        pos = plan["ranks"][r]
        xs = np.zeros((pos["counts"].sum(), d))
        for t in range(T_r):
            for j in range(k):
                xs[pos["dest_row"][t, j]] = [r, t, j, idx[r * T_r + t, j]]
        send.append(xs)
    recv_ref = ref.flat_all_to_all(send)
    for q in range(ep):
        recv = np.zeros_like(recv_ref[q])
        for r in range(ep):
            for t in range(T_r):
                for j in range(k):
                    if plan["owner"][r * T_r + t, j] == q:
                        recv[plan["recv_row"][r * T_r + t, j]] = [r, t, j, idx[r * T_r + t, j]]
        np.testing.assert_array_equal(recv, recv_ref[q])
    # involution: a2a . a2a = identity
    back = ref.flat_all_to_all(recv_ref)
    for r in range(ep):
        np.testing.assert_array_equal(back[r], send[r])

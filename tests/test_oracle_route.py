"""Pins of the oracle's route (F1) and route_bwd (B1) against brute force,
closed forms, library routines and invariants (CPU only)."""
import math

import numpy as np
import pytest
from scipy.special import softmax

import synth
from oracle import moe_ref as ref


def brute_topk(row, k):
    """Pure-Python: sort experts by (-value, index); NaN last; -0.0 == 0.0."""
    def key(e):
        v = float(row[e])
        if math.isnan(v):
            return (math.inf, e)
        return (-v + 0.0, e)
    return sorted(range(len(row)), key=key)[:k]


@pytest.mark.parametrize("E,k", [(8, 1), (8, 2), (64, 6), (256, 8), (5, 5)])
def test_topk_matches_brute_force(E, k):
    L = synth.random_logits(64, E, seed=E + k).numpy()
    # inject exact ties and signed zeros
    L[0, :] = 0.0
    L[1, ::2] = -0.0
    L[2, 3 % E] = L[2, 1 % E]
    idx = ref.topk_order(L, k)
    for t in range(L.shape[0]):
        assert list(idx[t]) == brute_topk(L[t], k)


def test_tie_fixture_all_zero_logits():
    """All-zero logits: experts 0..k-1 in order, gates exactly 1/k."""
    for E, k in [(8, 2), (64, 6), (256, 8)]:
        idx, g = ref.route(np.zeros((3, E), np.float32), k)
        assert (idx == np.arange(k)[None, :]).all()
        np.testing.assert_allclose(g, 1.0 / k, rtol=0, atol=1e-15)


def test_nan_sorts_below_minus_inf():
    L = np.array([[np.nan, -np.inf, 1.0, np.nan]], np.float32)
    idx = ref.topk_order(L, 4)
    assert list(idx[0]) == [2, 1, 0, 3]


def test_k_equals_E_is_full_sort():
    L = synth.random_logits(16, 8, seed=3).numpy()
    idx = ref.topk_order(L, 8)
    for t in range(16):
        assert list(idx[t]) == list(np.argsort(-L[t].astype(np.float64), kind="stable"))


def test_gates_sum_to_one_and_shift_invariant():
    L = synth.random_logits(128, 64, seed=11).numpy().astype(np.float64)
    idx, g = ref.route(L, 6)
    np.testing.assert_allclose(g.sum(1), 1.0, rtol=0, atol=4e-16)
    assert (np.diff(g, axis=1) <= 0).all()      # ordered by descending logit
    idx2, g2 = ref.route(L + 3.25, 6)
    assert (idx == idx2).all()
    np.testing.assert_allclose(g, g2, rtol=1e-13)


def test_gates_equal_softmax_then_renormalise():
    """Reading R1: softmax over the k selected == full softmax -> top-k -> renormalise
    (scipy's softmax is the library pin)."""
    L = synth.random_logits(50, 16, seed=5).numpy().astype(np.float64)
    idx, g = ref.route(L, 4)
    p = softmax(L, axis=1)
    sel = np.take_along_axis(p, idx.astype(np.int64), 1)
    np.testing.assert_allclose(g, sel / sel.sum(1, keepdims=True), rtol=1e-13)


def test_k1_gate_is_full_softmax_probability():
    L = synth.random_logits(40, 8, seed=9).numpy().astype(np.float64)
    idx, g = ref.route(L, 1)
    p = softmax(L, axis=1)
    np.testing.assert_allclose(g[:, 0], p[np.arange(40), idx[:, 0]], rtol=1e-13)
    assert (idx[:, 0] == np.argmax(L, axis=1)).all()


def test_column_permutation_equivariance():
    L = synth.random_logits(32, 16, seed=21).numpy()
    perm = np.random.default_rng(0).permutation(16)
    idx, g = ref.route(L, 3)
    idx_p, g_p = ref.route(L[:, perm], 3)
    assert (perm[idx_p] == idx).all()
    np.testing.assert_allclose(g, g_p, rtol=1e-14)


def test_topk_rejects_bad_k():
    with pytest.raises(ValueError):
        ref.topk_order(np.zeros((2, 4)), 5)
    with pytest.raises(ValueError):
        ref.topk_order(np.zeros((2, 4)), 0)


@pytest.mark.parametrize("k", [1, 2, 6])
def test_route_bwd_matches_finite_differences(k):
    """dl from route_bwd == central differences of sum_j g_j * dg_j (routing frozen)."""
    rng = np.random.default_rng(k)
    E = 8
    L = rng.standard_normal((6, E))
    idx, g = ref.route(L, k)
    dg = rng.standard_normal(g.shape)
    dl = ref.route_bwd(idx, g, dg, E, logits=L)
    h = 1e-6
    num = np.zeros_like(L)
    for t in range(L.shape[0]):
        for e in range(E):
            Lp, Lm = L.copy(), L.copy()
            Lp[t, e] += h
            Lm[t, e] -= h
            # freeze selection: evaluate gates at the original indices
            def gsum(M):
                sel = np.take_along_axis(M, idx.astype(np.int64), 1)
                if k == 1:
                    z = np.exp(M[t] - M[t].max())
                    return (z[idx[t, 0]] / z.sum()) * dg[t, 0]
                z = np.exp(sel[t] - sel[t].max())
                return float((z / z.sum()) @ dg[t])
            num[t, e] = (gsum(Lp) - gsum(Lm)) / (2 * h)
    np.testing.assert_allclose(dl, num, rtol=1e-6, atol=1e-8)
    if k > 1:
        np.testing.assert_allclose(dl.sum(1), 0.0, atol=1e-15)

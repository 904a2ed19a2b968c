"""Host-side model of the grouped GEMM's stream-K tail schedule (gemm.cu make_sched /
get_work, mirrored line by line) and its invariants over many launch shapes:

* every (tile, k-block) of the launch is computed by exactly one cluster, the data-parallel
  tiles whole and only the last partial wave split into k-chunks;
* a cluster takes all of its PARTIAL pieces before any FINISHING piece (so a partial
  producer never waits and the wait graph between clusters has no cycle);
* every partial slot is written once and read by exactly one finisher, the one holding the
  last k-chunk of the same tile;
* the split never makes the tail longer than the plain last wave.
"""
import math

import pytest


def make_sched(total, nkb, nc, c, enable=True, max_slots=336):
    rem_sk, S = 0, 1
    if enable:
        rem = total % nc
        best = (1, 1, 1)   # (S, rounds numerator, denominator)
        for s_ in (2, 3, 4):
            if rem == 0:
                break
            rounds = (s_ * rem + nc - 1) // nc
            if nkb // s_ >= 4 and (s_ - 1) * rem <= max_slots and rounds * best[2] < best[1] * s_:
                best = (s_, rounds, s_)
        if best[0] > 1:
            rem_sk, S = rem, best[0]
    dp = total - rem_sk
    n_dp = (dp - 1 - c) // nc + 1 if dp > c else 0
    pieces = S * rem_sk
    n_sk = (pieces - 1 - c) // nc + 1 if (S > 1 and pieces > c) else 0
    return dict(nc=nc, c=c, nkb=nkb, dp=dp, n_dp=n_dp, rem=rem_sk, S=S, n_sk=n_sk)


def get_work(s, w):
    """(tile, kb0, kb1, kind, slot(s))"""
    if w < s["n_dp"]:
        return s["c"] + w * s["nc"], 0, s["nkb"], "full", None
    p = s["c"] + (w - s["n_dp"]) * s["nc"]
    j, u = divmod(p, s["rem"])
    kb0, kb1 = j * s["nkb"] // s["S"], (j + 1) * s["nkb"] // s["S"]
    if j < s["S"] - 1:
        return s["dp"] + u, kb0, kb1, "partial", j * s["rem"] + u
    return s["dp"] + u, kb0, kb1, "finish", [jj * s["rem"] + u for jj in range(s["S"] - 1)]


@pytest.mark.parametrize("nc", [1, 2, 5, 64, 74, 148])
@pytest.mark.parametrize("nkb", [2, 3, 10, 32, 64, 224, 448])
def test_stream_k_schedule_invariants(nc, nkb):
    for total in list(range(1, 300, 7)) + [128, 160, 256, 448, 896]:
        cover, written, reads, per_cluster_pieces = {}, {}, {}, {}
        for c in range(nc):
            s = make_sched(total, nkb, nc, c)
            kinds, pieces = [], 0
            for w in range(s["n_dp"] + s["n_sk"]):
                t, kb0, kb1, kind, slot = get_work(s, w)
                kinds.append(kind)
                for kb in range(kb0, kb1):
                    assert (t, kb) not in cover
                    cover[(t, kb)] = c
                if kind == "partial":
                    assert slot not in written
                    written[slot] = t
                elif kind == "finish":
                    for sl in slot:
                        reads.setdefault(sl, []).append(t)
                if w >= s["n_dp"]:
                    pieces += 1
            sk_kinds = kinds[s["n_dp"]:]
            if "finish" in sk_kinds:
                first_finish = sk_kinds.index("finish")
                assert "partial" not in sk_kinds[first_finish:]
            per_cluster_pieces[c] = pieces
        assert len(cover) == total * nkb
        assert set(written) == set(reads)
        for sl, t in written.items():
            assert reads[sl] == [t]
        s0 = make_sched(total, nkb, nc, 0)
        if s0["S"] > 1:   # tail length in tiles: ceil(S rem / nc) / S < 1 (the plain last wave)
            assert math.ceil(s0["S"] * s0["rem"] / nc) < s0["S"]
            assert max(per_cluster_pieces.values()) == math.ceil(s0["S"] * s0["rem"] / nc)


def test_stream_k_only_for_a_poor_last_wave():
    # a full last wave keeps the plain data-parallel schedule
    assert make_sched(148, 64, 74, 0)["S"] == 1
    # Mixtral EP=8 GEMM2: 128 tiles on 74 clusters -> one data-parallel wave, then the 54
    # tail tiles in 4 k-chunks: 216 pieces in 3 rounds of a quarter tile (0.75 vs 1 wave)
    s = make_sched(128, 224, 74, 0)
    assert s["dp"] == 74 and s["rem"] == 54 and s["S"] == 4
    # EP=4 GEMM2: 256 tiles -> 34 tail tiles in halves, one round (0.5 wave)
    s = make_sched(256, 224, 74, 0)
    assert s["rem"] == 34 and s["S"] == 2

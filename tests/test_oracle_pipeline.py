"""Pins of the 1F1B schedule oracle (oracle/pipeline.py, reading R19)
against the paper's closed forms (PAPER.md:284 in-flight bound, PAPER.md:334-344 first/last
stage memory difference), the classic 1F1B makespan, and a dependency simulation; and the
libmoe schedule generator (moe_pipeline_1f1b, host code) against the oracle."""
import pytest

from oracle import pipeline as pl

CASES = [(pp, M) for pp in (1, 2, 3, 4, 8) for M in (1, 2, 3, 4, 7, 8, 16)]


@pytest.mark.parametrize("pp,M", CASES)
def test_each_stage_runs_every_microbatch_once_in_order(pp, M):
    for i in range(pp):
        ops = pl.schedule_1f1b(pp, i, M)
        assert [m for k, m in ops if k == pl.F] == list(range(M))
        assert [m for k, m in ops if k == pl.B] == list(range(M))
        for m in range(M):
            assert ops.index((pl.F, m)) < ops.index((pl.B, m))


@pytest.mark.parametrize("pp,M", CASES)
def test_peak_inflight_is_pp_minus_stage(pp, M):
    """stage i holds (PP - i) in-flight micro-batches at peak (at most M)."""
    for i in range(pp):
        assert pl.peak_inflight(pl.schedule_1f1b(pp, i, M)) == min(pp - i, M)


@pytest.mark.parametrize("pp,M", CASES)
def test_schedule_is_deadlock_free_with_the_1f1b_makespan(pp, M):
    """Unit-time forward and backward: the pipeline drains in 2 (M + PP - 1) ticks when
    M >= PP (bubble (PP - 1) / (M + PP - 1), Narayanan et al., cited at PAPER.md:126)."""
    ticks = pl.simulate(pp, M)
    assert len(ticks) == 2 * pp * M
    if M >= pp:
        assert max(ticks.values()) + 1 == 2 * (M + pp - 1)
    # stage 0's first backward waits for the whole pipeline: F goes down, B comes back
    assert ticks[(0, pl.B, 0)] == 2 * pp - 1


def test_first_and_last_stage_memory_difference():
    """M(0) - M(PP-1) = L (PP-1)/PP x (per-micro-batch activations); the
    expert-activation term of Eq. 4 with the in-flight counts of the schedule."""
    T_mb, ep, k, d, f, L = 4096, 2, 6, 2048, 1408, 8
    for pp in (2, 4):
        M = 8
        per = [pl.stage_activation_bytes(T_mb, ep, k, d, f, L // pp,
                                         pl.peak_inflight(pl.schedule_1f1b(pp, i, M)))
               for i in range(pp)]
        one_mb = 2 * (T_mb * k // ep) * (3 * f + d)
        assert per[0] - per[-1] == L * (pp - 1) // pp * one_mb
        assert per[0] == pp * per[-1]


@pytest.mark.parametrize("pp,M", CASES)
def test_libmoe_schedule_matches_the_oracle(pp, M):
    from paper_2605_05049_b200 import _lib as L
    for i in range(pp):
        assert L.moe_pipeline_1f1b(pp, i, M) == pl.schedule_1f1b(pp, i, M)


def test_libmoe_schedule_rejects_bad_arguments():
    from paper_2605_05049_b200 import _lib as L
    for args in [(0, 0, 4), (2, 2, 4), (2, -1, 4), (2, 0, 0)]:
        with pytest.raises(L.MoEError):
            L.moe_pipeline_1f1b(*args)

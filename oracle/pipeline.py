"""Oracle of the PP x EP pipelined executor.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product package.

PAPER.md:149 organises P GPUs into a PP x EP mesh: PP pipeline stages, each staffed by EP GPUs
that hold L/PP layers with their experts sharded E/EP per GPU; "there are EP
pipeline parallel groups of size PP and PP expert-parallel groups of size EP".  The executor
runs the 1F1B schedule (after Narayanan et al.): stage i holds at most
PP - i in-flight micro-batches.  Between stages, the EP GPU of the last layer
of stage i sends its activations to "its counterpart" in stage i+1.

Reading R19, the paper being silent on the exact op order: the PipeDream-flush
1F1B order -- stage i runs w = min(PP - i - 1, M) warm-up forwards, then alternates one forward
and one backward while forwards remain, then the remaining backwards; micro-batches in
ascending order in both directions.  Rank of mesh point (stage i, expert-parallel index e) is
i * EP + e (EP groups contiguous, the paper's "EP within the fast domain").

Pins (tests/test_oracle_pipeline.py, CPU): every micro-batch forwarded and backwarded once per
stage, F before B; peak in-flight = min(PP - i, M); a dependency simulation
drains without deadlock in 2 (M + PP - 1) unit ticks (the 1F1B makespan) with stage 0's first
backward at tick 2 PP - 1; M(0) - M(PP-1) = L (PP-1)/PP x one micro-batch's activations
(PAPER.md:334-344).
"""
from __future__ import annotations

F, B = 0, 1


def schedule_1f1b(pp, stage, M):
    """The op list of one stage: [(F|B, micro-batch), ...] (reading R19)."""
    if not (0 <= stage < pp) or M < 1:
        raise ValueError("need 0 <= stage < pp and M >= 1")
    w = min(pp - stage - 1, M)
    ops = [(F, m) for m in range(w)]
    nf, nb = w, 0
    while nf < M:
        ops.append((F, nf))
        nf += 1
        ops.append((B, nb))
        nb += 1
    while nb < M:
        ops.append((B, nb))
        nb += 1
    return ops


def peak_inflight(ops):
    """Largest number of micro-batches forwarded but not yet backwarded along an op list."""
    live = peak = 0
    for kind, _ in ops:
        live += 1 if kind == F else -1
        peak = max(peak, live)
    return peak


def simulate(pp, M):
    """Run every stage's op list against the data dependencies (F(i,m) needs F(i-1,m);
    B(i,m) needs B(i+1,m) and F(i,m)), one op per stage per tick when ready.  Returns the
    tick of every op {(stage, kind, m): tick}; raises on a deadlock."""
    lists = [schedule_1f1b(pp, i, M) for i in range(pp)]
    pos = [0] * pp
    done = {}
    tick = 0
    total = sum(len(l) for l in lists)
    while len(done) < total:
        fired = []
        for i in range(pp):
            if pos[i] == len(lists[i]):
                continue
            kind, m = lists[i][pos[i]]
            if kind == F:
                ready = i == 0 or (i - 1, F, m) in done
            else:
                ready = (i, F, m) in done and (i == pp - 1 or (i + 1, B, m) in done)
            if ready:
                fired.append((i, kind, m))
        if not fired:
            raise RuntimeError(f"1F1B deadlock at tick {tick}")
        for i, kind, m in fired:
            done[(i, kind, m)] = tick
            pos[i] += 1
        tick += 1
    return done


def stage_activation_bytes(T_mb, ep, k, d, f, layers_per_stage, inflight):
    """Eq. 4's expert-activation term per GPU of a stage (reading R16 of the
    saved tensors): inflight x L/PP x 2 (b/M) s k / EP x (3 d_ffn + d_model) bytes, with
    (b/M) s = T_mb tokens per micro-batch of the EP group; the attention terms of Eq. 4
    (12 b s d, 4 H b s^2) do not exist in an MoE-only stack."""
    return inflight * layers_per_stage * 2 * (T_mb * k // ep) * (3 * f + d)

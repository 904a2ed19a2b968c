"""Work counters of one MoE layer call, evaluated from the REALISED routing.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

These count what the layer actually does given a routing plan (rows per
expert, rows per (source, owner) pair).  Tests pin them against the paper's
closed forms on the balanced fixture ("6 FLOPs per parameter per
token"; PAPER.md:354-356 dispatch volumes; Table III / Eq. 2
activation and parameter bytes; PAPER.md:648 migration state 48 d f per
expert) -- the closed forms themselves live in the tests, not here.
"""
from __future__ import annotations

import numpy as np

BF16 = 2


def gemm_flops(expert_rows, d, f, T_local_shared=0, E_s=0):
    """Sum of 2*M*N*K over the expert GEMMs of one layer call.

    Forward per expert with n rows: X W_gate, X W_up (2 * 2 n d f) and H W_down
    (2 n f d) = 6 n d f.  Backward: dH = dO W_down^T (2 n d f), dX = [dG dU] [W_gate
    W_up]^T (4 n d f), dW_down = H^T dO (2 n f d), dW_gate|up = X^T [dG dU]
    (4 n d f) = 12 n d f.  Shared experts: the same on T_local_shared rows at
    width E_s*f.  Returns dict(fwd, bwd, total)."""
    n = int(np.sum(np.asarray(expert_rows, np.int64)))
    fwd = 6 * n * d * f + 6 * T_local_shared * d * (E_s * f)
    bwd = 2 * fwd
    return dict(fwd=fwd, bwd=bwd, total=fwd + bwd)


def router_flops(T, d, E):
    """F0 x W_r (2 T d E) and B0 dl W_r^T + x^T dl (4 T d E)."""
    return dict(fwd=2 * T * d * E, bwd=4 * T * d * E)


def pair_bytes(counts_all, d, ep):
    """NVLink bytes per (source r, owner q) for ONE all-to-all of bf16 rows:
    M[r, q] = d * 2 * sum_{e owned by q} counts_all[r, e].  The diagonal is the
    local (no-NVLink) part."""
    counts_all = np.asarray(counts_all, np.int64)
    EP, E = counts_all.shape
    E_l = E // ep
    per_owner = counts_all.reshape(EP, ep, E_l).sum(axis=2)
    return per_owner * d * BF16


def a2a_summary(counts_all, d, ep):
    """Per-rank egress/ingress (off-GPU) and send-buffer bytes for one a2a."""
    M = pair_bytes(counts_all, d, ep)
    off = M - np.diag(np.diag(M))
    return dict(pair=M, egress=off.sum(axis=1), ingress=off.sum(axis=0),
                send_buffer=M.sum(axis=1), total_off_gpu=int(off.sum()))


def expert_activation_bytes(expert_rows, d, f):
    """Saved expert activations of one rank: 2 bytes * rows * (3f + d)
    (G, U, H saved plus the expert input/output row; reading R10)."""
    return BF16 * int(np.sum(expert_rows)) * (3 * f + d)


def expert_state_bytes(n_experts, d, f, bytes_per_param=16):
    """Training state of n experts of 3 d f parameters at 16 B/param."""
    return bytes_per_param * 3 * n_experts * d * f


def hbm_bytes_permute(T_r, k_kept_rows, d):
    """F2 algorithmic HBM bytes: read x once (T_r d 2), write kept rows (rows d 2),
    plus the int32 index traffic (topk read, dest_row write)."""
    return BF16 * d * (T_r + k_kept_rows)


def hbm_bytes_unpermute(T_r, kept_rows, d):
    """F6 algorithmic HBM bytes: read kept rows, write y once."""
    return BF16 * d * (kept_rows + T_r)

"""fp64 oracle of the per-destination-rank deduplicated all-to-all.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product package.

What it computes.  The plain layer (moe_ref) sends one row per kept slot (t, j) to the
owner of expert e_{t,j}: a token whose k experts share an owner crosses NVLink several
times with the same bytes.  PAPER.md:119 credits X-MoE with "redundancy-based
communication bypassing" for exactly this; SURVEY.md §8(f) NEXT-4 names "per-destination-
rank token dedup" as the single-box variant of the paper's hierarchical all-to-all
(HALO, reduces to its Phase I inside one switch group).
Reading R18, step by step:

1. Pairs.  For source rank r, token t and owner q: (t, q) is a PAIR iff some kept slot j of
   t has owner(e_{t,j}) = q.  L_{r->q} = the pairs of r for q in ascending t;
   tslot[t, q] = index of t in L_{r->q} (-1 if not a pair); ntok[r][q] = |L_{r->q}|.
2. Dispatch.  x_t crosses once per pair into q's token buffer xt_q, rows ordered
   (source r, tslot): row = tok_base[q][r] + tslot, tok_base[q][r] = sum_{r'<r} ntok[r'][q].
   With it goes rlist[pair][j] = the receive row of slot (t, j) in q's expert-major buffer
   (moe_ref.dispatch_plan's recv_row, reading R7) if j is kept and owned by q, else -1,
   and glist[pair][j] = g_{t,j} under the same condition (else 0).
3. Expand (owner).  xr[rlist[u][j]] = xt[u] for every pair u and j with rlist >= 0: the
   same expert-major receive buffer as the plain dispatch, bit for bit.
4. Combine (owner -> source).  part[u] = sum_{j: rlist[u][j] >= 0} glist[u][j] * O[rlist[u][j]]
   (j ascending); it lands at the source's pair row pair_base[r][q] + tslot,
   pair_base[r][q] = sum_{q'<q} ntok[r][q'].  y_t = sum_q part[pair row of (t, q)] in
   ascending q (+ shared path).  Regrouping sum_j into sum_q sum_{j on q} is exact in real
   arithmetic; on the GPU the partials are rounded to bf16 once (a second rounding of y,
   inside the 2e-2 tolerance, reading R18).
5. Backward.  combine_bwd sends dy_t once per pair; the owner expands dO rows g*dy_t and
   forms dg_{t,j} = <dy_t, O_{t,j}> locally (O never leaves the owner); dispatch_bwd
   returns dxpart[u] = sum_{j on q} dX_{t,j} per pair, and dx_t = sum_q dxpart.

Pins (tests/test_oracle_dedup.py, CPU): pure-Python brute force of the pairs (also under a
migrated placement); the balanced-fixture closed form ntok[r][q] = max(1, k/E_l) T_r / EP and
the egress ratio; E_l = 1 or k = 1 reduce to the plain dispatch (one slot per pair, ntok =
counts per owner); invariants (every kept slot named exactly once, at moe_ref's receive row,
with its gate); expand rebuilds the plain receive buffer bit for bit; the pair reductions
reproduce moe_ref's y, dx and dgates to 1e-12; layout bases on a hand-worked matrix.
"""
from __future__ import annotations

import numpy as np


def pairs(dest_row_r, topk_idx_r, placement, E_l, ep):
    """Step 1 for one source rank.  dest_row_r [T_r,k] (-1 = dropped), topk_idx_r [T_r,k],
    placement[e] = global slot of expert e (owner = slot // E_l).
    Returns dict(owner [T_r,k], sent [T_r,EP] bool, tslot [T_r,EP] (-1 = no pair),
    ntok [EP])."""
    dest_row_r = np.asarray(dest_row_r, np.int64)
    idx = np.asarray(topk_idx_r, np.int64)
    placement = np.asarray(placement, np.int64)
    T_r, k = idx.shape
    owner = placement[idx] // E_l
    sent = np.zeros((T_r, ep), bool)
    t, j = np.nonzero(dest_row_r >= 0)
    sent[t, owner[t, j]] = True
    tslot = np.where(sent, np.cumsum(sent, axis=0) - 1, -1)
    return dict(owner=owner, sent=sent, tslot=tslot, ntok=sent.sum(axis=0).astype(np.int64))


def layout(ntok_all):
    """ntok_all [EP src, EP dst].  tok_base [q][r] = first row of source r in owner q's
    token buffer; tok_rows[q] = rows owner q receives; pair_base [r][q] = first pair row of
    owner q in source r's partial buffer; pair_rows[r] = pairs of source r."""
    n = np.asarray(ntok_all, np.int64)
    ep = n.shape[0]
    tok_base = np.zeros((ep, ep), np.int64)
    pair_base = np.zeros((ep, ep), np.int64)
    for q in range(ep):
        tok_base[q, 1:] = np.cumsum(n[:-1, q])
    for r in range(ep):
        pair_base[r, 1:] = np.cumsum(n[r, :-1])
    return dict(tok_base=tok_base, tok_rows=n.sum(axis=0), pair_base=pair_base,
                pair_rows=n.sum(axis=1))


def plan(topk_idx, gates, E, ep, C, align=1, placement=None):
    """Whole-EP-group dedup plan on top of moe_ref.dispatch_plan (steps 1-2).
    Returns dict(base = the plain plan, per-rank `pairs`, ntok_all, layout, and per owner q:
    rlist[q] [tok_rows[q], k], glist[q] [tok_rows[q], k], src[q] [tok_rows[q]] (source rank),
    tok[q] [tok_rows[q]] (global token index))."""
    from . import moe_ref as ref
    base = ref.dispatch_plan(topk_idx, E, ep, C, align, placement)
    placement = np.arange(E) if placement is None else np.asarray(placement, np.int64)
    T_r, E_l = base["T_r"], base["E_l"]
    topk_idx = np.asarray(topk_idx, np.int64)
    gates = np.asarray(gates, np.float64)
    k = topk_idx.shape[1]
    per = []
    for r in range(ep):
        sl = slice(r * T_r, (r + 1) * T_r)
        per.append(pairs(base["ranks"][r]["dest_row"], topk_idx[sl], placement, E_l, ep))
    ntok_all = np.stack([p["ntok"] for p in per])
    lay = layout(ntok_all)
    rlist, glist, src, tok = [], [], [], []
    for q in range(ep):
        n = int(lay["tok_rows"][q])
        rl = np.full((n, k), -1, np.int64)
        gl = np.zeros((n, k))
        sr = np.empty(n, np.int64)
        tk = np.empty(n, np.int64)
        for r in range(ep):
            p = per[r]
            ts = np.nonzero(p["sent"][:, q])[0]                  # ascending t = tslot order
            u = lay["tok_base"][q, r] + p["tslot"][ts, q]
            sr[u] = r
            tk[u] = r * T_r + ts
            for j in range(k):
                rows = base["recv_row"][r * T_r + ts, j]
                mine = (rows >= 0) & (p["owner"][ts, j] == q)
                rl[u[mine], j] = rows[mine]
                gl[u[mine], j] = gates[r * T_r + ts[mine], j]
        rlist.append(rl)
        glist.append(gl)
        src.append(sr)
        tok.append(tk)
    return dict(base=base, pairs=per, ntok_all=ntok_all, layout=lay, rlist=rlist, glist=glist,
                src=src, tok=tok, T_r=T_r, E_l=E_l, ep=ep, k=k)


def expand(xt, rlist, n_rows):
    """Step 3: xr [n_rows, d] with xr[rlist[u][j]] = xt[u]; rows no pair names stay zero
    (the padding rows of the 128-aligned receive segments)."""
    xt = np.asarray(xt)
    xr = np.zeros((n_rows, xt.shape[1]), dtype=xt.dtype)
    u, j = np.nonzero(rlist >= 0)
    xr[rlist[u, j]] = xt[u]
    return xr


def reduce_pairs(rows, rlist, glist=None):
    """Step 4 / 5 on one owner: part[u] = sum_j w[u][j] * rows[rlist[u][j]] over the pair's
    slots in j order, w = glist (combine) or 1 (dispatch_bwd).  fp64."""
    rows = np.asarray(rows, np.float64)
    n, k = rlist.shape
    part = np.zeros((n, rows.shape[1]))
    for j in range(k):
        m = rlist[:, j] >= 0
        w = 1.0 if glist is None else glist[m, j][:, None]
        part[m] += w * rows[rlist[m, j]]
    return part


def gather_pairs(parts_at_source, pr, pair_base):
    """Source side of steps 4 / 5: out_t = sum over owners q ascending of
    parts_at_source[pair_base[q] + tslot[t, q]] for every pair (t, q).  fp64."""
    parts = np.asarray(parts_at_source, np.float64)
    T_r, ep = pr["tslot"].shape
    out = np.zeros((T_r, parts.shape[1]))
    for q in range(ep):
        m = pr["tslot"][:, q] >= 0
        out[m] += parts[pair_base[q] + pr["tslot"][m, q]]
    return out


def egress_bytes(ntok_all, d, elem_bytes=2):
    """Per-rank off-GPU bytes of one dedup all-to-all: sum_{q != r} ntok[r][q] * d * 2
    (dispatch direction; the combine direction moves the same pair rows back)."""
    n = np.asarray(ntok_all, np.int64)
    return (n.sum(axis=1) - np.diag(n)) * d * elem_bytes

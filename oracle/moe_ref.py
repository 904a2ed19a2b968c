"""fp64 oracle of the expert-parallel MoE layer, step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the
product package; shares no code with it.

Notation follows PAPER.md Table II: d (hidden), E (routed
experts), E_s (shared experts), k (top-k), f = d_ffn^MoE, EP (expert-parallel
degree), T = b*s tokens of the whole EP group, T_r = T/EP tokens per rank.
Weights are in the paper's orientation:
    W_gate[e], W_up[e] in R^{d x f},  W_down[e] in R^{f x d},  W_r in R^{d x E}.

Everything floating is fp64 with no intermediate rounding (SURVEY.md §8(c)
c.3-9 reading: the paper's bf16 storage is absorbed by the tolerance).  The
discrete parts (top-k, capacity, positions, counts, rows) are exact.

Readings of points the paper leaves open are DESIGN.md "Readings" R1-R12; each
function names the ones it implements.
"""
from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# Elementwise functions of the SwiGLU expert (PAPER.md:229 names W_up, W_gate,
# W_down; reading R8: h = silu(x W_gate) * (x W_up), silu(z) = z*sigmoid(z)).
# ---------------------------------------------------------------------------


def sigmoid(z):
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def silu(z):
    return np.asarray(z, dtype=np.float64) * sigmoid(z)


def silu_grad(z):
    """d/dz silu(z) = sigmoid(z) * (1 + z*(1 - sigmoid(z)))."""
    s = sigmoid(z)
    return s * (1.0 + np.asarray(z, dtype=np.float64) * (1.0 - s))


# ---------------------------------------------------------------------------
# F0 router logits ("routing"; PAPER.md:50 learned gating)
# ---------------------------------------------------------------------------


def router_logits(x, W_r, bias=None):
    """l = x W_r (+ b).  x [T,d], W_r [d,E] -> [T,E] fp64.  The optional bias is
    the additive Zipf gate bias of the V3-like config (reading R11)."""
    L = np.asarray(x, np.float64) @ np.asarray(W_r, np.float64)
    if bias is not None:
        L = L + np.asarray(bias, np.float64)[None, :]
    return L


def router_logits_bwd(x, W_r, dlogits):
    """dx_router = dl W_r^T,  dW_r = x^T dl (per-rank partial; the EP all-reduce of
    dW_r is outside the layer, reading R12)."""
    dl = np.asarray(dlogits, np.float64)
    return dl @ np.asarray(W_r, np.float64).T, np.asarray(x, np.float64).T @ dl


# ---------------------------------------------------------------------------
# F1 route: top-k gating.
# Reading R1: gate = softmax over the k selected fp32 logits (k>1); k=1 keeps
#   the full-softmax probability of the chosen expert (Switch).
# Reading R2: ties go to the lower expert index, which is also ordered first;
#   -0.0 == +0.0; NaN sorts below -inf.
# Reading R3: selection on the fp32 logits (fp32 -> fp64 is exact).
# ---------------------------------------------------------------------------


def topk_order(logits, k):
    """Indices [T,k] of the k largest logits per row, sorted by the key
    (-l_{t,e}, e): descending value, ascending index among equal values."""
    L = np.asarray(logits, dtype=np.float64)
    T, E = L.shape
    if not 1 <= k <= E:
        raise ValueError(f"top-k needs 1 <= k <= E, got k={k}, E={E}")
    nan = np.isnan(L)                     # NaN below -inf: ordered last
    neg = np.where(nan, 0.0, -L) + 0.0    # -0.0 -> +0.0 (canonicalise)
    idx = np.broadcast_to(np.arange(E), L.shape)
    order = np.lexsort((idx, neg, nan), axis=-1)   # keys: isnan, then -l, then e
    return order[:, :k].astype(np.int32)


def route(logits, k):
    """Returns (topk_idx [T,k] int32, gates [T,k] fp64)."""
    L = np.asarray(logits, dtype=np.float64)
    idx = topk_order(L, k)
    sel = np.take_along_axis(L, idx.astype(np.int64), axis=1)
    if k == 1:
        # full softmax probability of the top expert: 1 / sum_e exp(l_e - l_0)
        z = np.exp(L - sel[:, :1])
        gates = 1.0 / z.sum(axis=1, keepdims=True)
    else:
        z = np.exp(sel - sel[:, :1])
        gates = z / z.sum(axis=1, keepdims=True)
    return idx, gates


def route_bwd(topk_idx, gates, dgates, E, logits=None):
    """dl[t, e_j] = g_j (dg_j - sum_i g_i dg_i), zero for unselected experts (k>1).
    For k=1 (full softmax): dl_e = dg * g0 * (delta_{e,e0} - p_e), needs logits."""
    topk_idx = np.asarray(topk_idx, np.int64)
    g = np.asarray(gates, np.float64)
    dg = np.asarray(dgates, np.float64)
    T, k = topk_idx.shape
    dl = np.zeros((T, E))
    if k == 1:
        L = np.asarray(logits, np.float64)
        p = np.exp(L - L.max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        dl = -(dg[:, :1] * g[:, :1]) * p
        np.put_along_axis(dl, topk_idx, np.take_along_axis(dl, topk_idx, 1) + dg * g, 1)
        return dl
    s = (g * dg).sum(axis=1, keepdims=True)
    np.put_along_axis(dl, topk_idx, g * (dg - s), axis=1)
    return dl


# ---------------------------------------------------------------------------
# F2 permute: capacity, positions, counts, dest_row (PAPER.md:129 token
# dropping; PAPER.md:231 per-expert token count s_e).
# Reading R4: C = ceil(cf*k*T_r/E) per (source rank, expert); cf <= 0: dropless.
# Reading R5: drop priority is slot-major, a = j*T_r + t (all first choices
#   before any second choice), then ascending local token index.
# Reading R6: gates are normalised over all k before dropping; a dropped slot
#   contributes 0 and is not renormalised away.
# ---------------------------------------------------------------------------


def capacity(cf, k, T_r, E):
    """C = ceil(cf*k*T_r/E) evaluated in fp64 from the fp32 value of cf (the capacity
    factor is an fp32 number of the problem statement, include/moe.h), or None
    (dropless) for cf <= 0.  E.g. cf=0.6 is 0.60000002384 in fp32: C(k=2,T=1500,E=8)=226."""
    cf32 = float(np.float32(cf))
    if cf32 <= 0:
        return None
    return int(math.ceil(cf32 * k * T_r / E))


def positions(topk_idx_r, E, C):
    """Per source rank.  p[t,j] = number of earlier assignments a' < a (a = j*T_r+t)
    with the same expert; kept = p < C; counts[e] = #kept; dest_row[t,j] =
    off[e] + p for kept slots (off = exclusive scan of counts), else -1.

    Returns dict(p, kept, counts, hist, off, dest_row)."""
    idx = np.asarray(topk_idx_r, np.int64)
    T_r, k = idx.shape
    flat = idx.T.reshape(-1)                     # slot-major order a = j*T_r + t
    order = np.argsort(flat, kind="stable")      # groups by expert, keeps a-order
    sorted_e = flat[order]
    hist = np.bincount(flat, minlength=E)
    first = np.concatenate(([0], np.cumsum(hist)[:-1]))
    p_flat = np.empty_like(flat)
    p_flat[order] = np.arange(flat.size) - first[sorted_e]
    p = p_flat.reshape(k, T_r).T
    kept = np.ones_like(p, dtype=bool) if C is None else p < C
    counts = hist if C is None else np.minimum(hist, C)
    off = np.concatenate(([0], np.cumsum(counts)[:-1]))
    dest_row = np.where(kept, off[idx] + p, -1)
    return dict(p=p, kept=kept, counts=counts.astype(np.int64), hist=hist.astype(np.int64),
                off=off.astype(np.int64), dest_row=dest_row.astype(np.int64))


def permute_rows(x_r, dest_row, n_rows):
    """xs[dest_row[t,j]] = x_t for kept slots.  Returns xs [n_rows, d]."""
    x_r = np.asarray(x_r)
    xs = np.zeros((n_rows, x_r.shape[1]), dtype=x_r.dtype)
    t, j = np.nonzero(dest_row >= 0)
    xs[dest_row[t, j]] = x_r[t]
    return xs


def permute_bwd(dxs, dest_row):
    """dx_t = sum_{j kept} dxs[dest_row[t,j]], accumulated in slot order j."""
    dxs = np.asarray(dxs, np.float64)
    T_r, k = dest_row.shape
    dx = np.zeros((T_r, dxs.shape[1]))
    for j in range(k):
        m = dest_row[:, j] >= 0
        dx[m] += dxs[dest_row[m, j]]
    return dx


# ---------------------------------------------------------------------------
# F3 dispatch placement ("each GPU gets E/EP experts").
# Reading R7: contiguous ownership, expert e on rank floor(e/E_l); receive rows
#   ordered (local expert, source rank, p); each local expert's rows form one
#   segment; segment starts are aligned to `align` rows (align=1 is the dense
#   canonical order; the kernels use align=128, include/moe.h).
# ---------------------------------------------------------------------------


def recv_layout(counts_all, ep, align=1, placement=None):
    """counts_all [EP, E] (kept rows from source r to expert e).  placement[e] = global slot
    of expert e (owner = slot // E_l, local slot = slot % E_l; default contiguous slot = e,
    reading R7; expert migration, NEXT-2, permutes it).  For owner q, per local slot el:
    recv_counts[q] [E_l, EP]; expert_rows[q] [E_l]; seg_base[q] [E_l+1] with
    seg_base[el+1] = seg_base[el] + roundup(expert_rows[el], align);
    src_base[q] [E_l, EP] = seg_base[el] + sum_{r'<r} counts[r'][e]; expert[q] [E_l]."""
    counts_all = np.asarray(counts_all, np.int64)
    EP, E = counts_all.shape
    if EP != ep or E % ep:
        raise ValueError("counts_all must be [EP, E] with EP | E")
    E_l = E // ep
    placement = np.arange(E) if placement is None else np.asarray(placement, np.int64)
    expert_at = np.empty(E, np.int64)
    expert_at[placement] = np.arange(E)
    out = []
    for q in range(ep):
        experts = expert_at[q * E_l:(q + 1) * E_l]
        rc = counts_all[:, experts].T.copy()                           # [E_l, EP]
        rows = rc.sum(axis=1)
        padded = -(-rows // align) * align
        seg = np.concatenate(([0], np.cumsum(padded)))
        src = seg[:-1, None] + np.concatenate((np.zeros((E_l, 1), np.int64),
                                               np.cumsum(rc, axis=1)[:, :-1]), axis=1)
        out.append(dict(recv_counts=rc, expert_rows=rows, seg_base=seg, src_base=src,
                        expert=experts))
    return out


def dispatch_plan(topk_idx, E, ep, C, align=1, placement=None):
    """Whole-EP-group routing plan.  topk_idx [T,k] global (rank r owns rows
    r*T_r..(r+1)*T_r-1).  Returns per-rank `positions` results, the [EP,E] count
    matrix, the receive layouts and recv_row[T,k] = row of slot (t,j) in its
    owner's receive buffer (-1 if dropped), owner[T,k]."""
    topk_idx = np.asarray(topk_idx, np.int64)
    T, k = topk_idx.shape
    if T % ep:
        raise ValueError("EP must divide T")
    T_r = T // ep
    E_l = E // ep
    ranks = [positions(topk_idx[r * T_r:(r + 1) * T_r], E, C) for r in range(ep)]
    counts_all = np.stack([r_["counts"] for r_ in ranks])
    placement = np.arange(E) if placement is None else np.asarray(placement, np.int64)
    layouts = recv_layout(counts_all, ep, align, placement)
    owner = placement[topk_idx] // E_l
    recv_row = np.full((T, k), -1, np.int64)
    for r in range(ep):
        pos = ranks[r]
        sl = slice(r * T_r, (r + 1) * T_r)
        e = topk_idx[sl]
        q = placement[e] // E_l
        el = placement[e] % E_l
        base = np.empty_like(e)
        for qq in range(ep):
            m = q == qq
            base[m] = layouts[qq]["src_base"][el[m], r]
        recv_row[sl] = np.where(pos["kept"], base + pos["p"], -1)
    return dict(T_r=T_r, E_l=E_l, ranks=ranks, counts_all=counts_all, layouts=layouts,
                recv_row=recv_row, owner=owner)


# ---------------------------------------------------------------------------
# F4 expert FFN and its backward (n_mat = 3 SwiGLU)
# ---------------------------------------------------------------------------


def expert_forward(X, W_gate, W_up, W_down):
    """G = X W_gate, U = X W_up, H = silu(G)*U, O = H W_down."""
    X = np.asarray(X, np.float64)
    G = X @ np.asarray(W_gate, np.float64)
    U = X @ np.asarray(W_up, np.float64)
    H = silu(G) * U
    O = H @ np.asarray(W_down, np.float64)
    return G, U, H, O


def expert_backward(X, G, U, H, dO, W_gate, W_up, W_down):
    """dH = dO W_down^T; dG = dH*U*silu'(G); dU = dH*silu(G);
    dX = dG W_gate^T + dU W_up^T; dW_down = H^T dO; dW_gate = X^T dG; dW_up = X^T dU."""
    X = np.asarray(X, np.float64)
    dO = np.asarray(dO, np.float64)
    dH = dO @ np.asarray(W_down, np.float64).T
    dG = dH * U * silu_grad(G)
    dU = dH * silu(G)
    dX = dG @ np.asarray(W_gate, np.float64).T + dU @ np.asarray(W_up, np.float64).T
    return dict(dX=dX, dW_down=H.T @ dO, dW_gate=X.T @ dG, dW_up=X.T @ dU, dG=dG, dU=dU, dH=dH)


# ---------------------------------------------------------------------------
# Whole layer (all EP ranks simulated in one process), given fp32 logits.
# F5 combine returns O rows to their source row; F6 y_t = sum_{j kept}
# g_{t,j} O_{t,j} + SharedFFN(x_t)  (reading R9 shared experts: unweighted,
# local; E_s experts of width f == one SwiGLU of width E_s*f).
# ---------------------------------------------------------------------------


def moe_forward(x, logits, W_gate, W_up, W_down, k, cf, ep, shared=None):
    """x [T,d] (global), logits [T,E] fp32 (teacher-forced routing boundary),
    W_* lists/arrays indexed by expert in paper orientation,
    shared = (W_gate_s [d,E_s f], W_up_s, W_down_s [E_s f, d]) or None.
    Returns a dict holding y [T,d] and everything backward needs."""
    x = np.asarray(x, np.float64)
    T, d = x.shape
    E = np.asarray(logits).shape[1]
    if E % ep or T % ep:
        raise ValueError("EP must divide E and T")
    topk_idx, gates = route(logits, k)
    C = capacity(cf, k, T // ep, E)
    plan = dispatch_plan(topk_idx, E, ep, C)
    kept = plan["recv_row"] >= 0
    O_slots = np.zeros((T, k, d))
    cache = {}
    for e in range(E):
        t, j = np.nonzero((topk_idx == e) & kept)
        if t.size == 0:
            cache[e] = None
            continue
        # rows of expert e in receive order (source rank, p) == ascending recv_row
        order = np.argsort(plan["recv_row"][t, j], kind="stable")
        t, j = t[order], j[order]
        G, U, H, O = expert_forward(x[t], W_gate[e], W_up[e], W_down[e])
        O_slots[t, j] = O
        cache[e] = (t, j, G, U, H)
    g_kept = np.where(kept, gates, 0.0)
    y = np.einsum("tj,tjd->td", g_kept, O_slots)
    sh = None
    if shared is not None:
        Gs, Us, Hs, Os = expert_forward(x, *shared)
        y = y + Os
        sh = (Gs, Us, Hs)
    return dict(y=y, x=x, logits=np.asarray(logits, np.float64), topk_idx=topk_idx,
                gates=gates, C=C, plan=plan, kept=kept, O_slots=O_slots, cache=cache,
                shared=shared, shared_cache=sh, k=k, E=E, ep=ep)


def moe_backward(fw, dy, W_gate, W_up, W_down):
    """Backward of moe_forward given dy [T,d].  Returns dict(dx_experts, dgates,
    dlogits, dW_gate, dW_up, dW_down (lists per expert, zero for empty experts),
    dx_shared, dW_gate_s, dW_up_s, dW_down_s)."""
    dy = np.asarray(dy, np.float64)
    x, kept, gates = fw["x"], fw["kept"], fw["gates"]
    T, d = x.shape
    E = fw["E"]
    dgates = np.where(kept, np.einsum("td,tjd->tj", dy, fw["O_slots"]), 0.0)
    dx = np.zeros((T, d))
    dWg, dWu, dWd = [], [], []
    for e in range(E):
        c = fw["cache"][e]
        if c is None:
            dWg.append(np.zeros_like(np.asarray(W_gate[e], np.float64)))
            dWu.append(np.zeros_like(np.asarray(W_up[e], np.float64)))
            dWd.append(np.zeros_like(np.asarray(W_down[e], np.float64)))
            continue
        t, j, G, U, H = c
        dO = gates[t, j][:, None] * dy[t]
        b = expert_backward(x[t], G, U, H, dO, W_gate[e], W_up[e], W_down[e])
        np.add.at(dx, t, b["dX"])
        dWg.append(b["dW_gate"])
        dWu.append(b["dW_up"])
        dWd.append(b["dW_down"])
    out = dict(dx_experts=dx, dgates=dgates, dW_gate=dWg, dW_up=dWu, dW_down=dWd)
    out["dlogits"] = route_bwd(fw["topk_idx"], gates, dgates, E, logits=fw["logits"])
    if fw["shared"] is not None:
        Gs, Us, Hs = fw["shared_cache"]
        b = expert_backward(x, Gs, Us, Hs, dy, *fw["shared"])
        out.update(dx_shared=b["dX"], dW_gate_s=b["dW_gate"], dW_up_s=b["dW_up"],
                   dW_down_s=b["dW_down"])
    else:
        out["dx_shared"] = np.zeros((T, d))
    return out


def layer_forward_backward(x, W_r, W_gate, W_up, W_down, dy, k, cf, ep, shared=None,
                           bias=None, logits=None):
    """Full layer incl. router: logits (fp64 unless given), MoE forward, backward,
    dx = experts + shared + router terms; dW_r = sum over ranks of x_r^T dl_r."""
    L = router_logits(x, W_r, bias) if logits is None else logits
    fw = moe_forward(x, L, W_gate, W_up, W_down, k, cf, ep, shared)
    bw = moe_backward(fw, dy, W_gate, W_up, W_down)
    dx_r, dW_r = router_logits_bwd(x, W_r, bw["dlogits"])
    bw["dx"] = bw["dx_experts"] + bw["dx_shared"] + dx_r
    bw["dW_r"] = dW_r
    return fw, bw


# ---------------------------------------------------------------------------
# All-to-all reference (SPEC.md:467-503 functional a2a; transpose law).
# ---------------------------------------------------------------------------


def flat_all_to_all(send):
    """send[r] is rank r's buffer split into EP equal chunks (chunk q -> rank q).
    recv[q] chunk r = send[r] chunk q (brute-force N^2 copy)."""
    ep = len(send)
    chunks = [np.split(np.asarray(s), ep) for s in send]
    return [np.concatenate([chunks[r][q] for r in range(ep)]) for q in range(ep)]

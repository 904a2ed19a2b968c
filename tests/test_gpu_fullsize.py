"""Full-size parity (BASELINE.json shapes) on one GPU, in the launch configuration bench.py
times, on outputs the oracle can compute one by one:

* routing, capacity positions, counts and the receive layout: ALL tokens, bit-exact;
* y, dx and dgates: a seeded sample of 512 tokens (SURVEY.md §8(c) c.5 CI mode), each
  computed by the oracle from that token alone (its kept experts' full SwiGLU forward, the
  per-token backward, the router term), per tensor and per token row;
* weight gradients: the FULL dW_gate, dW_up, dW_down of 4 experts (the most loaded and 3
  seeded others), over all of each expert's rows.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import moe_ref as ref
from tests.helpers import TOL, expected_dest_row, f64, paper_weights, rel_err, rel_err_rows

pytestmark = pytest.mark.gpu

# SURVEY.md §8(c) c.5 CI mode: 512 tokens per rank for y / dx / dgates, and the FULL weight
# gradients of 4 experts (the most loaded one and 3 seeded others)
N_TOK, N_EXPERTS = 512, 4


@pytest.mark.parametrize("name", ["mixtral", "dsmoe", "dsv3"])
def test_fullsize_sampled_parity(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.test_gpu_layer import build_layer
    cfg = synth.CONFIGS[name]
    layer = build_layer(cfg)                      # EP=1, all experts on this GPU
    x = synth.tokens(cfg, device="cuda")
    dy = synth.grad_output(cfg, device="cuda")
    y = layer.forward(x).clone()
    dx = layer.backward(dy).clone()
    torch.cuda.synchronize()
    layer.ctx.check_device_error()

    # ---- discrete parts, all tokens
    logits = layer.logits.cpu().numpy()
    idx, gates = ref.route(logits, cfg.k)
    assert (layer.topk_idx.cpu().numpy() == idx).all()
    C = ref.capacity(cfg.cf, cfg.k, cfg.T, cfg.E)
    plan = ref.dispatch_plan(idx, cfg.E, 1, C, align=128)
    pos = plan["ranks"][0]
    assert (layer.counts.cpu().numpy() == pos["counts"]).all()
    assert (layer.dest_row.cpu().numpy() == expected_dest_row(layer, idx, C, cfg.E)).all()
    lay = layer.layout.cpu().numpy()
    assert (lay[cfg.E:2 * cfg.E] == plan["layouts"][0]["expert_rows"]).all()
    assert (lay[2 * cfg.E:] == plan["layouts"][0]["seg_base"]).all()
    assert rel_err(f64(layer.gates), gates) < 1e-5

    # ---- sampled tokens: y, dx, dgates; the oracle runs each expert on the sampled slots
    # routed to it (a token's result depends only on its own row)
    rng = np.random.default_rng(0)
    toks = np.sort(rng.choice(cfg.T, N_TOK, replace=False))
    kept = pos["dest_row"] >= 0
    xs, dys = f64(x[toks]), f64(dy[toks])
    w_r = f64(layer.w_r).T
    y_ref = np.zeros((N_TOK, cfg.d))
    dx_ref = np.zeros((N_TOK, cfg.d))
    dg = np.zeros((N_TOK, cfg.k))
    sel = idx[toks]
    ksel = kept[toks]
    for e in sorted(set(sel[ksel].tolist())):   # one expert at a time (bounded memory)
        i, j = np.nonzero((sel == e) & ksel)
        Wg, Wu, Wd = paper_weights(layer.w_gu[e], layer.w_down[e], cfg.f)
        G, U, H, O = ref.expert_forward(xs[i], Wg, Wu, Wd)
        g = gates[toks[i], j][:, None]
        np.add.at(y_ref, i, g * O)
        dg[i, j] = np.einsum("nd,nd->n", dys[i], O)
        b = ref.expert_backward(xs[i], G, U, H, g * dys[i], Wg, Wu, Wd)
        np.add.at(dx_ref, i, b["dX"])
    if cfg.E_s:
        Sg, Su, Sd = paper_weights(layer.w_gu_s, layer.w_down_s, cfg.E_s * cfg.f)
        G, U, H, O = ref.expert_forward(xs, Sg, Su, Sd)
        y_ref += O
        dx_ref += ref.expert_backward(xs, G, U, H, dys, Sg, Su, Sd)["dX"]
    dl = ref.route_bwd(idx[toks], gates[toks], dg, cfg.E, logits=logits[toks])
    dx_ref += ref.router_logits_bwd(xs, w_r, dl)[0]
    errs = {"y": rel_err(f64(y[toks]), y_ref), "dx": rel_err(f64(dx[toks]), dx_ref),
            "dgates": rel_err(f64(layer.dgates[toks]), dg),
            "y_rows": rel_err_rows(f64(y[toks]), y_ref),
            "dx_rows": rel_err_rows(f64(dx[toks]), dx_ref),
            "dgates_rows": rel_err_rows(f64(layer.dgates[toks]), dg)}

    # ---- full weight gradients of N_EXPERTS experts (all their rows, all columns)
    rows_e = plan["layouts"][0]["expert_rows"]
    hot = int(np.argmax(rows_e))
    others = [int(e) for e in rng.permutation(cfg.E) if e != hot][:N_EXPERTS - 1]
    for e in [hot] + others:
        t_e, j_e = np.nonzero((idx == e) & kept)
        if t_e.size == 0:
            assert (f64(layer.dw_gu[e]) == 0).all()
            continue
        order = np.argsort(pos["dest_row"][t_e, j_e], kind="stable")
        t_e, j_e = t_e[order], j_e[order]
        Wg, Wu, Wd = paper_weights(layer.w_gu[e], layer.w_down[e], cfg.f)
        ti = torch.from_numpy(t_e).cuda()
        Xe = f64(x[ti])
        dOe = gates[t_e, j_e][:, None] * f64(dy[ti])
        G, U, H, _ = ref.expert_forward(Xe, Wg, Wu, Wd)
        b = ref.expert_backward(Xe, G, U, H, dOe, Wg, Wu, Wd)
        dgu = f64(layer.dw_gu[e])
        errs[f"dW_gate{e}"] = rel_err(dgu[:cfg.f].T, b["dW_gate"])
        errs[f"dW_up{e}"] = rel_err(dgu[cfg.f:].T, b["dW_up"])
        errs[f"dW_down{e}"] = rel_err(f64(layer.dw_down[e]).T, b["dW_down"])
        del G, U, H, b
    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if not v < TOL}
    assert not bad, bad
    layer.close()

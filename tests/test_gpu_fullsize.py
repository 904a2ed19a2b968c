"""Full-size parity (BASELINE.json shapes) on one GPU, in the launch configuration bench.py
times, on outputs the oracle can compute one by one:

* routing, capacity positions, counts and the receive layout: ALL tokens, bit-exact;
* y and dx: a seeded sample of tokens, each computed by the oracle from that token alone
  (its kept experts' full SwiGLU forward, the per-token backward, the router term);
* weight gradients: for two experts, a seeded sample of f-columns -- SwiGLU columns are
  independent, so the oracle's expert_backward on the column-restricted expert gives
  exactly those columns of dW_gate, dW_up and rows of dW_down over all the expert's rows.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import moe_ref as ref
from tests.helpers import TOL, f64, paper_weights, rel_err

pytestmark = pytest.mark.gpu

SAMPLES = {"mixtral": (48, 64), "dsmoe": (48, 64), "dsv3": (12, 64)}


@pytest.mark.parametrize("name", ["mixtral", "dsmoe", "dsv3"])
def test_fullsize_sampled_parity(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.test_gpu_layer import build_layer
    cfg = synth.CONFIGS[name]
    n_tok, n_col = SAMPLES[name]
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
    assert (layer.dest_row.cpu().numpy() == pos["dest_row"]).all()
    lay = layer.layout.cpu().numpy()
    assert (lay[cfg.E:2 * cfg.E] == plan["layouts"][0]["expert_rows"]).all()
    assert (lay[2 * cfg.E:] == plan["layouts"][0]["seg_base"]).all()
    assert rel_err(f64(layer.gates), gates) < 1e-5

    # ---- sampled tokens: y and dx computed token by token
    rng = np.random.default_rng(0)
    toks = np.sort(rng.choice(cfg.T, n_tok, replace=False))
    kept = pos["dest_row"] >= 0
    xs, dys = f64(x[toks]), f64(dy[toks])
    w_r = f64(layer.w_r).T
    y_ref = np.zeros((n_tok, cfg.d))
    dx_ref = np.zeros((n_tok, cfg.d))
    dg = np.zeros((n_tok, cfg.k))
    need = sorted(set(idx[toks][kept[toks]].tolist()))
    cache = {}
    for e in need:   # one expert at a time (bounded memory)
        Wg, Wu, Wd = paper_weights(layer.w_gu[e], layer.w_down[e], cfg.f)
        for i, t in enumerate(toks):
            for j in range(cfg.k):
                if kept[t, j] and idx[t, j] == e:
                    G, U, H, O = ref.expert_forward(xs[i:i + 1], Wg, Wu, Wd)
                    y_ref[i] += gates[t, j] * O[0]
                    dg[i, j] = float(dys[i] @ O[0])
                    b = ref.expert_backward(xs[i:i + 1], G, U, H, gates[t, j] * dys[i:i + 1],
                                            Wg, Wu, Wd)
                    dx_ref[i] += b["dX"][0]
    if cfg.E_s:
        Sg, Su, Sd = paper_weights(layer.w_gu_s, layer.w_down_s, cfg.E_s * cfg.f)
        G, U, H, O = ref.expert_forward(xs, Sg, Su, Sd)
        y_ref += O
        dx_ref += ref.expert_backward(xs, G, U, H, dys, Sg, Su, Sd)["dX"]
    dl = ref.route_bwd(idx[toks], gates[toks], dg, cfg.E, logits=logits[toks])
    dx_ref += ref.router_logits_bwd(xs, w_r, dl)[0]
    e_y = rel_err(f64(y[toks]), y_ref)
    e_dx = rel_err(f64(dx[toks]), dx_ref)
    e_dg = rel_err(f64(layer.dgates[toks]), dg)

    # ---- weight gradients of two experts on sampled f-columns (all rows of the expert)
    errs = {}
    rows_e = plan["layouts"][0]["expert_rows"]
    for e in [int(np.argmax(rows_e)), int(rng.integers(0, cfg.E))]:
        t_e, j_e = np.nonzero((idx == e) & kept)
        if t_e.size == 0:
            continue
        order = np.argsort(pos["dest_row"][t_e, j_e], kind="stable")
        t_e, j_e = t_e[order], j_e[order]
        cols = np.sort(rng.choice(cfg.f, n_col, replace=False))
        Wg, Wu, Wd = paper_weights(layer.w_gu[e], layer.w_down[e], cfg.f)
        Xe = f64(x[torch.from_numpy(t_e).cuda()])
        dOe = gates[t_e, j_e][:, None] * f64(dy[torch.from_numpy(t_e).cuda()])
        G, U, H, _ = ref.expert_forward(Xe, Wg[:, cols], Wu[:, cols], Wd[cols, :])
        b = ref.expert_backward(Xe, G, U, H, dOe, Wg[:, cols], Wu[:, cols], Wd[cols, :])
        dgu = layer.dw_gu[e]
        errs[f"dW_gate{e}"] = rel_err(f64(dgu[torch.from_numpy(cols).cuda()]).T, b["dW_gate"])
        errs[f"dW_up{e}"] = rel_err(f64(dgu[torch.from_numpy(cols + cfg.f).cuda()]).T, b["dW_up"])
        errs[f"dW_down{e}"] = rel_err(f64(layer.dw_down[e][:, torch.from_numpy(cols).cuda()]).T,
                                      b["dW_down"])
    errs.update(y=e_y, dx=e_dx, dgates=e_dg)
    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if not v < TOL}
    assert not bad, bad
    layer.close()

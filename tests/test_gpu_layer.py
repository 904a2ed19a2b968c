"""End-to-end parity of one MoE layer (forward + backward) at EP=1 through the C ABI
against the fp64 oracle, given the GPU's fp32 logits as
the routing boundary (the oracle recomputes nothing discrete from its own logits)."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import moe_ref as ref
from tests.helpers import TOL, expected_dest_row, f64, paper_weights, rel_err, rel_err_rows

pytestmark = pytest.mark.gpu

CASES = {
    "tiny": synth.CONFIGS["tiny"],
    "mixtral_small": synth.MoEConfig("mixtral_small", T=1024, d=512, E=8, k=2, f=1024, cf=1.25),
    "dsmoe_small": synth.MoEConfig("dsmoe_small", T=1024, d=256, E=64, k=6, f=128, cf=1.25, E_s=2),
    "v3_small_zipf": synth.MoEConfig("v3_small_zipf", T=2048, d=512, E=256, k=8, f=256, cf=0.0,
                                     zipf_s=1.0),
    "drops": synth.MoEConfig("drops", T=600, d=128, E=8, k=2, f=256, cf=0.5),
    # k = 1 (Switch-style): dense router gradient -> the GEMM path of moe_router_logits_bwd
    "switch_k1": synth.MoEConfig("switch_k1", T=512, d=128, E=8, k=1, f=256, cf=1.25),
}


def build_layer(cfg, ep_size=1, ep_rank=0, device=0, dedup=False, **kw):
    from paper_2605_05049_b200 import LayerDims, MoELayer
    T_r = cfg.T // ep_size
    dims = LayerDims(T_r, cfg.d, cfg.E, cfg.k, cfg.f, cfg.E_s, cfg.cf, ep_size, ep_rank)
    layer = MoELayer(dims, device=device, dedup=dedup, **kw)
    E_l = cfg.E // ep_size
    experts = range(ep_rank * E_l, (ep_rank + 1) * E_l)
    dev = torch.device(f"cuda:{device}")
    # weights drawn on the GPU (the CUDA generator is deterministic per seed), as bench.py does
    w_gu, w_down = synth.expert_weights(cfg, experts, device=dev)
    w_gu_s, w_down_s = synth.shared_weights(cfg, device=dev)
    layer.set_weights(synth.router_weight(cfg, device=dev), w_gu, w_down, synth.zipf_bias(cfg),
                      w_gu_s, w_down_s)
    return layer


def oracle_layer(cfg, x, dy, logits, ep=1):
    """The fp64 oracle on the same inputs (weights re-drawn from the same CUDA seeds)."""
    w_r = f64(synth.router_weight(cfg, device="cuda")).T
    w_gu, w_down = synth.expert_weights(cfg, range(cfg.E), device="cuda")
    Wg, Wu, Wd = [], [], []
    for e in range(cfg.E):
        a, b, c = paper_weights(w_gu[e], w_down[e], cfg.f)
        Wg.append(a); Wu.append(b); Wd.append(c)
    shared = None
    if cfg.E_s:
        s_gu, s_down = synth.shared_weights(cfg, device="cuda")
        shared = paper_weights(s_gu, s_down, cfg.E_s * cfg.f)
    fw, bw = ref.layer_forward_backward(f64(x), w_r, Wg, Wu, Wd, f64(dy), cfg.k, cfg.cf, ep,
                                        shared=shared, logits=logits)
    return fw, bw


@pytest.mark.parametrize("name,dedup", [(n, False) for n in CASES] +
                         [(n, m) for n in ("mixtral_small", "dsmoe_small", "v3_small_zipf",
                                           "drops") for m in ("dispatch", "all")])
def test_layer_ep1_parity(name, dedup):
    """dedup: the NEXT-4 deduplicated all-to-alls (reading R18) on the same checks, plus the
    pair tables bit-exact against oracle/dedup.py and xr bitwise equal to the plain dispatch's
    receive buffer; mode "dispatch" must also give the plain layer's outputs bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CASES[name]
    layer = build_layer(cfg, dedup=dedup)
    x = synth.tokens(cfg).cuda()
    dy = synth.grad_output(cfg).cuda()
    y = layer.forward(x).clone()
    dx = layer.backward(dy).clone()
    torch.cuda.synchronize()
    layer.ctx.check_device_error()
    logits = layer.logits.cpu().numpy()
    # router logits vs fp64 (fp32 accumulation of bf16 products)
    want_l = ref.router_logits(f64(x), f64(layer.w_r).T,
                               None if synth.zipf_bias(cfg) is None else f64(synth.zipf_bias(cfg)))
    assert np.abs(logits - want_l).max() < 1e-3
    fw, bw = oracle_layer(cfg, x, dy, logits)
    # discrete parts: bit-exact
    assert (layer.topk_idx.cpu().numpy() == fw["topk_idx"]).all()
    pos = fw["plan"]["ranks"][0]
    assert (layer.counts.cpu().numpy() == pos["counts"]).all()
    assert (layer.dest_row.cpu().numpy() == expected_dest_row(layer, fw["topk_idx"], fw["C"],
                                                              cfg.E)).all()
    lay = layer.layout.cpu().numpy()
    E_l = cfg.E
    assert (lay[:cfg.E] == fw["plan"]["counts_all"][0]).all()
    assert (lay[cfg.E:cfg.E + E_l] == fw["plan"]["layouts"][0]["expert_rows"]).all()
    if dedup:
        from oracle import dedup as dd
        P = dd.plan(fw["topk_idx"], fw["gates"], cfg.E, 1, fw["C"], align=128)
        assert (layer.pdest.cpu().numpy() == P["pairs"][0]["tslot"]).all()   # EP=1: pair_base 0
        assert (layer.ntok.cpu().numpy() == P["ntok_all"][0]).all()
        assert (layer.dlayout.cpu().numpy() == P["ntok_all"].reshape(-1)).all()
        n = int(P["layout"]["tok_rows"][0])
        assert (layer.rlist[:n].cpu().numpy() == P["rlist"][0]).all()
        gl = layer.glist[:n].cpu().numpy()
        assert (gl == layer.gates.cpu().numpy()[P["tok"][0]] * (P["rlist"][0] >= 0)).all()
        # the expanded receive buffer is the plain dispatch's, bit for bit (128-aligned layout)
        base = P["base"]
        xr = layer.xr.cpu()
        t, j = np.nonzero(base["recv_row"] >= 0)
        assert torch.equal(xr[torch.as_tensor(base["recv_row"][t, j])], x.cpu()[torch.as_tensor(t)])
        n_rows = int(lay[cfg.E + E_l + E_l])
        pad = np.ones(n_rows, bool)
        pad[base["recv_row"][t, j]] = False
        assert (xr[:n_rows][torch.as_tensor(pad)] == 0).all()
    if dedup == "dispatch":
        plain = build_layer(cfg)
        yp = plain.forward(x).clone()
        dxp = plain.backward(dy).clone()
        torch.cuda.synchronize()
        assert torch.equal(yp, y) and torch.equal(dxp, dx)
        assert torch.equal(plain.dgates, layer.dgates) and torch.equal(plain.dw_gu, layer.dw_gu)
        assert torch.equal(plain.dw_down, layer.dw_down) and torch.equal(plain.dw_r, layer.dw_r)
        plain.close()
    # floating parts within tolerance
    errs = {}
    errs["gates"] = rel_err(f64(layer.gates), fw["gates"])
    errs["y"] = rel_err(f64(y), fw["y"])
    errs["dgates"] = rel_err(f64(layer.dgates), bw["dgates"])
    errs["dlogits"] = rel_err(f64(layer.dlogits), bw["dlogits"])
    errs["dx"] = rel_err(f64(dx), bw["dx"])
    errs["dW_r"] = rel_err(f64(layer.dw_r).T, bw["dW_r"])
    # per token row as well (a wrong small row cannot hide behind the tensor's largest one)
    errs["y_rows"] = rel_err_rows(f64(y), fw["y"])
    errs["dx_rows"] = rel_err_rows(f64(dx), bw["dx"])
    errs["dgates_rows"] = rel_err_rows(f64(layer.dgates), bw["dgates"])
    # (dlogits: per tensor only -- each row is k-sparse and a difference g_j (dg_j - sum g dg),
    # so its per-row scale is set by cancellation; the dgates rows it is formed from are checked)
    for e in range(cfg.E):
        if fw["cache"][e] is None:
            assert (f64(layer.dw_gu[e]) == 0).all() and (f64(layer.dw_down[e]) == 0).all()
            continue
        dgu = f64(layer.dw_gu[e])
        errs[f"dW_gate{e}"] = rel_err(dgu[:cfg.f].T, bw["dW_gate"][e])
        errs[f"dW_up{e}"] = rel_err(dgu[cfg.f:].T, bw["dW_up"][e])
        errs[f"dW_down{e}"] = rel_err(f64(layer.dw_down[e]).T, bw["dW_down"][e])
    if cfg.E_s:
        fs = cfg.E_s * cfg.f
        dgs = f64(layer.dw_gu_s[0])
        errs["dW_gate_s"] = rel_err(dgs[:fs].T, bw["dW_gate_s"])
        errs["dW_up_s"] = rel_err(dgs[fs:].T, bw["dW_up_s"])
        errs["dW_down_s"] = rel_err(f64(layer.dw_down_s[0]).T, bw["dW_down_s"])
    worst = max(errs, key=errs.get)
    print(f"{name}: worst {worst} = {errs[worst]:.2e}; y {errs['y']:.2e} dx {errs['dx']:.2e}")
    bad = {k: v for k, v in errs.items() if not v < TOL}
    assert not bad, bad
    layer.close()


def test_identity_experts_and_determinism():
    """FFN bypassed (dispatch -> combine with out = xr): y = (sum_{j kept} g) x within one
    bf16 rounding; two identical calls are bit-identical."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_05049_b200 import _lib as L
    cfg = CASES["drops"]
    layer = build_layer(cfg)
    x = synth.tokens(cfg).cuda()
    c = layer.ctx
    L.moe_router_logits(c, x, layer.w_r, None, layer.logits)
    L.moe_route(c, layer.logits, layer.topk_idx, layer.gates)
    L.moe_permute(c, x, layer.topk_idx, layer.counts, layer.dest_row, layer.xs)
    L.moe_dispatch(c, layer.xs, layer.counts, layer.layout, layer.xr)
    L.moe_combine(c, layer.xr, layer.layout, layer.ys, layer.gates, layer.dest_row, None, layer.y)
    torch.cuda.synchronize()
    y1 = layer.y.clone()
    kept = (layer.dest_row >= 0).float()
    gs = (layer.gates * kept).sum(1, keepdim=True)
    want = (gs * x.float()).to(torch.bfloat16)
    diff = (y1.float() - want.float()).abs()
    ulp = want.float().abs() * 2.0 ** -7 + 1e-30
    assert (diff <= ulp).all()
    # determinism of the whole layer
    dy = synth.grad_output(cfg).cuda()
    ya = layer.forward(x).clone(); dxa = layer.backward(dy).clone(); dwa = layer.dw_gu.clone()
    yb = layer.forward(x).clone(); dxb = layer.backward(dy).clone(); dwb = layer.dw_gu.clone()
    torch.cuda.synchronize()
    assert torch.equal(ya, yb) and torch.equal(dxa, dxb) and torch.equal(dwa, dwb)
    layer.close()


@pytest.mark.parametrize("name", ["mixtral_small", "dsmoe_small", "drops"])
def test_fused_and_stepwise_paths_bit_identical(name):
    """moe_expert_ffn_combine / moe_expert_ffn_bwd_dispatch (GEMM epilogues storing rows
    straight into the sources' buffers) give bit-identical y, dx and weight gradients to
    the step-by-step moe_expert_ffn + moe_combine / moe_expert_ffn_bwd + moe_dispatch_bwd."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CASES[name]
    x = synth.tokens(cfg).cuda()
    dy = synth.grad_output(cfg).cuda()
    outs = []
    for fused in (True, False):
        layer = build_layer(cfg)
        layer.fused = fused
        y = layer.forward(x).clone()
        dx = layer.backward(dy).clone()
        torch.cuda.synchronize()
        layer.ctx.check_device_error()
        outs.append((y, dx, layer.dw_gu.clone(), layer.dw_down.clone(), layer.dgates.clone()))
        layer.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("name", ["v3_small_zipf", "dsmoe_small"])
def test_expert_placement_is_bit_identical(name):
    """Expert migration (NEXT-2): after migrate() to a random placement (experts in other
    slots, weights moved with them) the layer's y, dx and every expert's weight gradient are
    bit-identical to the contiguous placement, and the layout record equals the oracle's
    placement-aware receive layout."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CASES[name]
    layer = build_layer(cfg)
    x = synth.tokens(cfg).cuda()
    dy = synth.grad_output(cfg).cuda()
    y0 = layer.forward(x).clone()
    dx0 = layer.backward(dy).clone()
    gu0, dn0 = layer.dw_gu.clone(), layer.dw_down.clone()
    perm = np.random.default_rng(5).permutation(cfg.E)
    assert layer.migrate(perm) == 0          # EP = 1: slots move, nothing crosses ranks
    y1 = layer.forward(x).clone()
    dx1 = layer.backward(dy).clone()
    torch.cuda.synchronize()
    layer.ctx.check_device_error()
    assert torch.equal(y0, y1) and torch.equal(dx0, dx1)
    for slot, e in enumerate(layer.experts_of_slots()):
        assert torch.equal(layer.dw_gu[slot], gu0[e]) and torch.equal(layer.dw_down[slot], dn0[e])
    idx = layer.topk_idx.cpu().numpy()
    plan = ref.dispatch_plan(idx, cfg.E, 1, ref.capacity(cfg.cf, cfg.k, cfg.T, cfg.E), align=128,
                             placement=perm)
    lay = layer.layout.cpu().numpy()
    assert (lay[cfg.E:2 * cfg.E] == plan["layouts"][0]["expert_rows"]).all()
    assert (lay[2 * cfg.E:] == plan["layouts"][0]["seg_base"]).all()
    layer.close()


@pytest.mark.parametrize("name", ["mixtral_small", "dsmoe_small"])
def test_graph_replay_bit_identical(name):
    """MoELayer.capture: the fwd+bwd step replayed from a CUDA graph equals the eager step bit
    for bit, and a replay after overwriting the captured input equals the eager step on it."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CASES[name]
    layer = build_layer(cfg)
    x = synth.tokens(cfg).cuda()
    dy = synth.grad_output(cfg).cuda()
    y0 = layer.forward(x).clone()
    dx0 = layer.backward(dy).clone()
    gu0 = layer.dw_gu.clone()
    xg, dyg = x.clone(), dy.clone()
    g = layer.capture(xg, dyg)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(layer.y, y0) and torch.equal(layer.dx, dx0)
        assert torch.equal(layer.dw_gu, gu0)
    x2 = synth.tokens(cfg, seed=11).cuda()
    xg.copy_(x2)
    g.replay()
    y2g, dx2g = layer.y.clone(), layer.dx.clone()
    y2 = layer.forward(x2).clone()
    dx2 = layer.backward(dy).clone()
    torch.cuda.synchronize()
    layer.ctx.check_device_error()
    assert torch.equal(y2g, y2) and torch.equal(dx2g, dx2) and not torch.equal(y2, y0)
    layer.close()


@pytest.mark.parametrize("dedup", [False, "dispatch"])
def test_empty_token_shard(dedup):
    """T_local = 0 is legal (include/moe.h): every call is a no-op that still takes part in the
    collectives -- forward and backward complete, weight gradients are exactly zero, dx and y
    are empty, the layout record shows zero rows, and the device error word stays clear."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = synth.MoEConfig("empty", T=0, d=256, E=8, k=2, f=256, cf=1.25, E_s=1)
    layer = build_layer(cfg, dedup=dedup)
    x = torch.empty((0, cfg.d), dtype=torch.bfloat16, device="cuda")
    for _ in range(2):
        y = layer.forward(x)
        dx = layer.backward(x)
    torch.cuda.synchronize()
    layer.ctx.check_device_error()
    assert y.shape == (0, cfg.d) and dx.shape == (0, cfg.d)
    assert int(layer.layout.abs().sum().item()) == 0
    assert (layer.dw_gu == 0).all() and (layer.dw_down == 0).all() and (layer.dw_r == 0).all()
    assert (layer.dw_gu_s == 0).all() and (layer.dw_down_s == 0).all()
    layer.close()


@pytest.mark.parametrize("name", ["mixtral_small", "dsmoe_small", "drops", "v3_small_zipf"])
def test_ep1_local_path_bit_identical(name):
    """EP = 1 local path (moe_permute_dispatch_local: the permute writes the 128-aligned
    receive layout itself) against moe_permute + moe_dispatch: the layout record,
    xr (incl. zeroed padding), y, dx and every weight gradient bit for bit -- also under a
    migrated slot placement."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CASES[name]
    x = synth.tokens(cfg).cuda()
    dy = synth.grad_output(cfg).cuda()
    perm = np.random.default_rng(3).permutation(cfg.E)
    for place in (None, perm):
        outs = []
        for fast in (True, False):
            layer = build_layer(cfg)
            layer.local_fast_path = fast
            if place is not None:
                layer.migrate(place)
            layer.xr.fill_(3.0)          # stale rows must be overwritten or zeroed
            y = layer.forward(x).clone()
            dx = layer.backward(dy).clone()
            torch.cuda.synchronize()
            layer.ctx.check_device_error()
            n = int(layer.layout[-1].item())
            outs.append((y, dx, layer.dw_gu.clone(), layer.dw_down.clone(), layer.layout.clone(),
                         layer.xr[:n].clone()))
            layer.close()
        for a, b in zip(*outs):
            assert torch.equal(a, b)


@pytest.mark.parametrize("name", ["mixtral_small", "dsmoe_small", "drops", "v3_small_zipf"])
def test_tile_overlap_bit_identical(name):
    """NEXT-1 tile-granular overlap -- moe_dispatch_expert_ffn_up (the dispatch inside the GEMM1
    launch) and moe_combine_bwd_expert_ffn_dh (combine_bwd inside dgrad-1), tiles gated by
    per-(slot, source) arrival flags -- against the separate transfer + GEMM calls on the
    general path at EP = 1 (the transfers then target this rank's own heap): layout record,
    xr and dO incl. zeroed padding, G|U|H, dG|dU, dgates, y, dx and the weight gradients bit
    for bit, over repeated steps (the flag epochs and the work counters must reset) and under
    a migrated placement."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CASES[name]
    x = synth.tokens(cfg).cuda()
    dy = synth.grad_output(cfg).cuda()
    perm = np.random.default_rng(5).permutation(cfg.E)
    for place in (None, perm):
        outs = []
        for tile in (True, False):
            layer = build_layer(cfg)
            layer.local_fast_path = False
            layer.tile_overlap = layer.tile_overlap_bwd = tile
            if place is not None:
                layer.migrate(place)
            for step in range(3):
                layer.xr.fill_(3.0)          # stale rows must be overwritten or zeroed
                layer.dout_r.fill_(7.0)
                layer.g_u_h.fill_(5.0)
                y = layer.forward(x).clone()
                dx = layer.backward(dy).clone()
                torch.cuda.synchronize()
                layer.ctx.check_device_error()
                n = int(layer.layout[-1].item())
                outs.append((y, dx, layer.dw_gu.clone(), layer.dw_down.clone(),
                             layer.layout.clone(), layer.xr[:n].clone(), layer.g_u_h[:n].clone(),
                             layer.dgates.clone(), layer.dout_r[:n].clone(), layer.dgu[:n].clone()))
            layer.close()
        ref = outs[0]
        for o in outs[1:]:
            for a, b in zip(ref, o):
                assert torch.equal(a, b)

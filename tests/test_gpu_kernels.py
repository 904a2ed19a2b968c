"""Per-step parity of the CUDA path (through the C ABI) against the fp64 oracle.

Teacher-forced: each step is fed the GPU's own inputs to
that step, cast exactly to fp64, and compared with the oracle step.  Discrete
outputs (indices, counts, positions, rows) must be bit-exact; floating outputs
within helpers.TOL."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import moe_ref as ref
from tests.helpers import TOL, f64, paper_weights, rel_err, seg_bases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_05049_b200 import _lib
    return _lib


def make_ctx(L, T, d, E, k, f, cf=1.25, E_s=0, heap=1 << 20):
    shape = L.make_shape(T, d, E, k, f, E_s, cf, 1, 0)
    return L.Context(shape, 0, heap), shape


# ---------------------------------------------------------------- F1 route
@pytest.mark.parametrize("T,E,k", [(256, 8, 2), (1000, 64, 6), (777, 256, 8), (64, 8, 1), (33, 5, 5)])
def test_route_bit_exact(L, T, E, k):
    ctx, _ = make_ctx(L, T, 64, E, k, 128)
    logits = synth.random_logits(T, E, seed=T + E).cuda()
    logits[0] = 0.0                     # full tie -> experts 0..k-1
    logits[1, ::2] = -0.0               # signed zeros tie with +0.0
    logits[2, :] = torch.arange(E, dtype=torch.float32).cuda() % 3   # repeated values
    idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
    g = torch.empty((T, k), dtype=torch.float32, device="cuda")
    L.moe_route(ctx, logits, idx, g)
    torch.cuda.synchronize()
    ref_idx, ref_g = ref.route(logits.cpu().numpy(), k)
    assert (idx.cpu().numpy() == ref_idx).all()
    np.testing.assert_allclose(g.cpu().numpy(), ref_g, rtol=2e-6, atol=1e-7)
    ctx.close()


def test_route_bwd(L):
    T, E, k = 300, 64, 6
    ctx, _ = make_ctx(L, T, 64, E, k, 128)
    logits = synth.random_logits(T, E, seed=3).cuda()
    idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
    g = torch.empty((T, k), dtype=torch.float32, device="cuda")
    L.moe_route(ctx, logits, idx, g)
    dg = synth.random_logits(T, k, seed=4).cuda()
    dl = torch.empty((T, E), dtype=torch.float32, device="cuda")
    L.moe_route_bwd(ctx, logits, idx, g, dg, dl)
    torch.cuda.synchronize()
    ref_dl = ref.route_bwd(idx.cpu().numpy(), f64(g), f64(dg), E)
    assert rel_err(f64(dl), ref_dl) < 1e-5
    ctx.close()


# ---------------------------------------------------------------- F2 permute / B2 / F6
@pytest.mark.parametrize("T,E,k,cf", [(256, 8, 2, 1.25), (2048, 64, 6, 1.25), (1500, 8, 2, 0.6),
                                      (4096, 256, 8, 0.0), (37, 8, 2, 1.0)])
def test_permute_bit_exact(L, T, E, k, cf):
    d = 128
    ctx, shape = make_ctx(L, T, d, E, k, 128, cf=cf)
    x = synth.tokens(synth.CONFIGS["tiny"], T=T).cuda()
    x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    logits = synth.random_logits(T, E, seed=11).cuda()
    if cf > 0 and cf < 1:
        logits[:, 0] += 1.0            # skew -> capacity drops
    idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
    g = torch.empty((T, k), dtype=torch.float32, device="cuda")
    L.moe_route(ctx, logits, idx, g)
    counts = torch.empty((E,), dtype=torch.int32, device="cuda")
    dest = torch.empty((T, k), dtype=torch.int32, device="cuda")
    xs = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    L.moe_permute(ctx, x, idx, counts, dest, xs)
    torch.cuda.synchronize()
    C = ref.capacity(cf, k, T, E)
    assert L.moe_capacity(shape) == (-1 if C is None else C)
    pos = ref.positions(idx.cpu().numpy(), E, C)
    assert (counts.cpu().numpy() == pos["counts"]).all()
    assert (dest.cpu().numpy() == pos["dest_row"]).all()
    n = int(pos["counts"].sum())
    xs_ref = ref.permute_rows(x.cpu().view(torch.int16).numpy(), pos["dest_row"], n)
    assert (xs[:n].cpu().view(torch.int16).numpy() == xs_ref).all()      # bitwise rows
    # permute_bwd with unit rows: dx = round_bf16(n_kept * x) bitwise (exact fp32 sum)
    dx = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    L.moe_permute_bwd(ctx, xs, dest, None, None, dx)
    torch.cuda.synchronize()
    n_kept = torch.from_numpy(pos["kept"].sum(1)).cuda().float()[:, None]
    assert torch.equal(dx, (n_kept * x.float()).to(torch.bfloat16))
    ctx.close()


def test_unpermute_and_extras(L):
    T, E, k, d = 512, 8, 2, 256
    ctx, _ = make_ctx(L, T, d, E, k, 128)
    logits = synth.random_logits(T, E, seed=5).cuda()
    idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
    g = torch.empty((T, k), dtype=torch.float32, device="cuda")
    L.moe_route(ctx, logits, idx, g)
    x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    counts = torch.empty((E,), dtype=torch.int32, device="cuda")
    dest = torch.empty((T, k), dtype=torch.int32, device="cuda")
    xs = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    L.moe_permute(ctx, x, idx, counts, dest, xs)
    acc = torch.randn((T, d), device="cuda")
    extra = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    dx = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    L.moe_permute_bwd(ctx, xs, dest, acc, extra, dx)
    torch.cuda.synchronize()
    kept = (dest >= 0).float().sum(1, keepdim=True)
    want = kept.double().cpu() * f64(x) + f64(acc) + f64(extra)
    assert rel_err(f64(dx), want) < 8e-3
    ctx.close()


# ---------------------------------------------------------------- F0 router logits
@pytest.mark.parametrize("T,d,E", [(256, 64, 8), (1000, 2048, 64), (300, 7168, 256), (129, 512, 8)])
def test_router_logits(L, T, d, E):
    ctx, _ = make_ctx(L, T, d, E, 2, 128)
    cfg = synth.MoEConfig("t", T=T, d=d, E=E, k=2, f=128, cf=1.25)
    x = synth.tokens(cfg).cuda()
    w_r = synth.router_weight(cfg).cuda()
    bias = torch.randn(E, device="cuda")
    logits = torch.empty((T, E), dtype=torch.float32, device="cuda")
    L.moe_router_logits(ctx, x, w_r, bias, logits)
    torch.cuda.synchronize()
    want = ref.router_logits(f64(x), f64(w_r).T, f64(bias))
    # fp32 accumulation of bf16 products: absolute error ~ sqrt(d) * 2^-24 * |x||w|
    assert np.abs(f64(logits) - want).max() < 1e-4 * max(1.0, math.sqrt(d / 64))
    ctx.close()


@pytest.mark.parametrize("T,d,E", [(500, 1024, 64), (8192, 4096, 8), (300, 7168, 256), (77, 64, 5)])
def test_router_bwd(L, T, d, E):
    ctx, _ = make_ctx(L, T, d, E, 2, 128)
    cfg = synth.MoEConfig("t", T=T, d=d, E=E, k=2, f=128, cf=1.25)
    x = synth.tokens(cfg).cuda()
    w_r = synth.router_weight(cfg).cuda()
    dl = synth.random_logits(T, E, seed=9).cuda()
    dx = torch.empty((T, d), dtype=torch.float32, device="cuda")
    dw = torch.empty((E, d), dtype=torch.float32, device="cuda")
    L.moe_router_logits_bwd(ctx, x, w_r, dl, dx, dw, False)
    torch.cuda.synchronize()
    rdx, rdw = ref.router_logits_bwd(f64(x), f64(w_r).T, f64(dl))
    # dl enters the tensor cores as bf16 hi + lo (|dl - hi - lo| <= 2^-17 |dl|)
    assert rel_err(f64(dx), rdx) < 1e-4
    assert rel_err(f64(dw), rdw.T) < 1e-4
    # accumulate adds onto the previous dW_r
    L.moe_router_logits_bwd(ctx, x, w_r, dl, None, dw, True)
    torch.cuda.synchronize()
    assert rel_err(f64(dw), 2 * rdw.T) < 1e-4
    ctx.close()


@pytest.mark.parametrize("T,d,E,k", [(1000, 512, 8, 2), (700, 1024, 64, 6), (300, 7168, 256, 8)])
def test_permute_bwd_router_fused(L, T, d, E, k):
    """B2 + B0-dgrad fused (k-sparse router gradient) == oracle dx = sum dxs rows + dl W_r^T."""
    ctx, _ = make_ctx(L, T, d, E, k, 128, cf=1.0)
    cfg = synth.MoEConfig("t", T=T, d=d, E=E, k=k, f=128, cf=1.0)
    w_r = synth.router_weight(cfg).cuda()
    logits = synth.random_logits(T, E, seed=21).cuda()
    idx = torch.empty((T, k), dtype=torch.int32, device="cuda")
    g = torch.empty((T, k), dtype=torch.float32, device="cuda")
    L.moe_route(ctx, logits, idx, g)
    x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    counts = torch.empty((E,), dtype=torch.int32, device="cuda")
    dest = torch.empty((T, k), dtype=torch.int32, device="cuda")
    xs = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    L.moe_permute(ctx, x, idx, counts, dest, xs)          # xs doubles as a dxs stand-in
    dg = synth.random_logits(T, k, seed=22).cuda()
    dl = torch.empty((T, E), dtype=torch.float32, device="cuda")
    L.moe_route_bwd(ctx, logits, idx, g, dg, dl)
    extra = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    dx = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    L.moe_permute_bwd_router(ctx, xs, dest, idx, dl, w_r, extra, dx)
    torch.cuda.synchronize()
    pos = ref.positions(idx.cpu().numpy(), E, ref.capacity(1.0, k, T, E))
    want = ref.permute_bwd(f64(xs), pos["dest_row"])
    want += ref.router_logits_bwd(f64(x), f64(w_r).T, f64(dl))[0] + f64(extra)
    assert rel_err(f64(dx), want) < 8e-3
    # the dense path gives the same numbers: dx_router GEMM + moe_permute_bwd(dx_acc)
    dxr = torch.empty((T, d), dtype=torch.float32, device="cuda")
    L.moe_router_logits_bwd(ctx, x, w_r, dl, dxr, None, False)
    dx2 = torch.empty_like(dx)
    L.moe_permute_bwd(ctx, xs, dest, dxr, extra, dx2)
    torch.cuda.synchronize()
    assert rel_err(f64(dx2), f64(dx)) < 8e-3
    ctx.close()


# ---------------------------------------------------------------- F4 / B4 grouped expert FFN
def _ffn_case(rows, d, f, seed=0):
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    seg = seg_bases(rows)
    R = int(seg[-1]) + 128
    xr = torch.zeros((R, d), dtype=torch.bfloat16)
    for i, n in enumerate(rows):
        xr[seg[i]:seg[i] + n] = torch.randn((n, d), generator=g).to(torch.bfloat16)
    G = len(rows)
    w_gu = (torch.randn((G, 2 * f, d), generator=g) / math.sqrt(d)).to(torch.bfloat16)
    w_down = (torch.randn((G, d, f), generator=g) / math.sqrt(f)).to(torch.bfloat16)
    return seg, R, xr, w_gu, w_down


@pytest.mark.parametrize("rows,d,f", [([100, 0, 300, 128], 256, 256), ([513], 64, 128),
                                      ([37, 1, 200], 512, 384), ([1024, 999], 2048, 1408)])
def test_expert_ffn_fwd_bwd(L, rows, d, f):
    seg, R, xr, w_gu, w_down = _ffn_case(rows, d, f)
    G = len(rows)
    ctx, _ = make_ctx(L, 128, d, 8, 2, f)
    xr_d, w_gu_d, w_down_d = xr.cuda(), w_gu.cuda(), w_down.cuda()
    gr = torch.tensor(rows, dtype=torch.int32, device="cuda")
    g_u_h = torch.full((R, 3 * f), float("nan"), dtype=torch.bfloat16, device="cuda")
    out = torch.full((R, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    L.moe_expert_ffn(ctx, xr_d, gr, G, R, f, w_gu_d, w_down_d, g_u_h, out)
    torch.cuda.synchronize()
    dout = torch.zeros((R, d), dtype=torch.bfloat16)
    for i, n in enumerate(rows):
        dout[seg[i]:seg[i] + n] = torch.randn((n, d)).to(torch.bfloat16)
    dout_d = dout.cuda()
    dgu = torch.empty((R, 2 * f), dtype=torch.bfloat16, device="cuda")
    dxr = torch.empty((R, d), dtype=torch.bfloat16, device="cuda")
    dw_gu = torch.full((G, 2 * f, d), float("nan"), dtype=torch.float32, device="cuda")
    dw_down = torch.full((G, d, f), float("nan"), dtype=torch.float32, device="cuda")
    L.moe_expert_ffn_bwd(ctx, xr_d, gr, G, R, f, w_gu_d, w_down_d, g_u_h, dout_d, dgu, dxr, dw_gu,
                         dw_down, False)
    torch.cuda.synchronize()
    ghu = f64(g_u_h)
    for i, n in enumerate(rows):
        s0, s1 = int(seg[i]), int(seg[i + 1])
        Wg, Wu, Wd = paper_weights(w_gu[i], w_down[i], f)
        X = f64(xr[s0:s0 + n])
        Gr, Ur, Hr, Or = ref.expert_forward(X, Wg, Wu, Wd)
        if n:
            assert rel_err(ghu[s0:s0 + n, :f], Gr) < TOL, ("G", i)
            assert rel_err(ghu[s0:s0 + n, f:2 * f], Ur) < TOL, ("U", i)
            assert rel_err(ghu[s0:s0 + n, 2 * f:], Hr) < TOL, ("H", i)
            assert rel_err(f64(out[s0:s0 + n]), Or) < TOL, ("O", i)
        # padding rows inside the segment are zero
        assert (ghu[s0 + n:s1] == 0).all() and (f64(out[s0 + n:s1]) == 0).all()
        # backward, teacher-forced from the GPU's saved G,U,H
        Gs, Us, Hs = ghu[s0:s0 + n, :f], ghu[s0:s0 + n, f:2 * f], ghu[s0:s0 + n, 2 * f:]
        b = ref.expert_backward(X, Gs, Us, Hs, f64(dout[s0:s0 + n]), Wg, Wu, Wd)
        dgu_h = f64(dgu)
        if n:
            assert rel_err(dgu_h[s0:s0 + n, :f], b["dG"]) < TOL, ("dG", i)
            assert rel_err(dgu_h[s0:s0 + n, f:], b["dU"]) < TOL, ("dU", i)
            assert rel_err(f64(dxr[s0:s0 + n]), b["dX"]) < TOL, ("dX", i)
            # wgrad vs the oracle fed with the GPU's dG, dU (teacher forcing)
            assert rel_err(f64(dw_down[i]), (Hs.T @ f64(dout[s0:s0 + n])).T) < TOL, ("dWd", i)
            dGU = dgu_h[s0:s0 + n]
            assert rel_err(f64(dw_gu[i]), dGU.T @ X) < TOL, ("dWgu", i)
        else:
            assert (f64(dw_gu[i]) == 0).all() and (f64(dw_down[i]) == 0).all()
    # accumulate=True adds
    before = dw_down.clone()
    L.moe_expert_ffn_bwd(ctx, xr_d, gr, G, R, f, w_gu_d, w_down_d, g_u_h, dout_d, dgu, dxr, dw_gu,
                         dw_down, True)
    torch.cuda.synchronize()
    assert torch.allclose(dw_down, 2 * before, rtol=1e-6, atol=1e-6)
    ctx.close()

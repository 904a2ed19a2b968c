"""torchrun worker: one EP rank per GPU runs the MoE layer on its token shard and its
experts (NVSwitch peer-store dispatch/combine); rank 0 gathers everything and checks it
against the fp64 oracle simulating all EP ranks (tests/test_gpu_multi.py launches it).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tests/mp_layer_worker.py --config tiny
Prints one JSON line on rank 0: {"ok": bool, "errors": {...}, ...}.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from tests import mp_common  # noqa: E402

CASES = {
    "tiny": synth.MoEConfig("tiny_ep", T=512, d=64, E=8, k=2, f=128, cf=1.25),
    "mixtral_small": synth.MoEConfig("mixtral_small", T=2048, d=512, E=8, k=2, f=1024, cf=1.25),
    "dsmoe_small": synth.MoEConfig("dsmoe_small", T=2048, d=256, E=64, k=6, f=128, cf=1.25, E_s=2),
    "v3_small_zipf": synth.MoEConfig("v3_small_zipf", T=2048, d=512, E=256, k=8, f=256, cf=0.0,
                                     zipf_s=1.0),
    "drops": synth.MoEConfig("drops", T=1024, d=128, E=8, k=2, f=256, cf=0.5),
    # one expert per rank at nproc 4 (the Mixtral EP=8 layout, E_l = 1, on 4 GPUs)
    "el1": synth.MoEConfig("el1", T=2048, d=512, E=4, k=2, f=1024, cf=1.25),
    # expert collapse: a strong Zipf bias sends every token to two experts, so
    # most ranks receive no rows at all (empty GEMM groups) and send everything away
    "collapse": synth.MoEConfig("collapse", T=512, d=128, E=8, k=2, f=256, cf=0.0, zipf_s=8.0),
    # T_local = 0 on every rank: the collectives still run (include/moe.h)
    "empty": synth.MoEConfig("empty", T=0, d=128, E=8, k=2, f=256, cf=1.25, E_s=1),
}


gather = mp_common.gather


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny", choices=list(CASES))
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--stepwise", action="store_true", help="unfused step-by-step calls")
    ap.add_argument("--rebalance", action="store_true",
                    help="observe loads, run Alg. 2 (moe_rebalance) and migrate before checking")
    ap.add_argument("--dedup", nargs="?", const="dispatch", default=None,
                    choices=["dispatch", "all"],
                    help="NEXT-4 deduplicated all-to-alls (pair tables and xr checked bitwise)")
    ap.add_argument("--graph", action="store_true",
                    help="also replay the step from a CUDA graph (device-side collective epoch)")
    args = ap.parse_args()
    local, shared = mp_common.init()
    ep, rank = dist.get_world_size(), dist.get_rank()
    cfg = CASES[args.config]
    from tests.test_gpu_layer import build_layer, oracle_layer
    from tests.helpers import TOL, f64, rel_err, rel_err_rows

    n_par = 3 * cfg.d * cfg.f                       # parameters per expert
    layer = build_layer(cfg, ep_size=ep, ep_rank=rank, device=local, dedup=args.dedup,
                        expert_state_bytes=3 * 4 * n_par if args.rebalance else 0)
    E_l = cfg.E // ep
    code = lambda e: (e + (torch.arange(n_par, device="cuda") % 7).float() / 8)   # exact in fp32
    if args.rebalance:
        # optimizer-like state (fp32 master copy + two moments: the 12 of the paper's 16 B per
        # parameter) registered to move with the experts
        opt = [layer.expert_state(nm, (n_par,), torch.float32) for nm in ("master", "m", "v")]
        for i, t in enumerate(opt):
            for el in range(E_l):
                t[el].copy_(code(rank * E_l + el) * (i + 1))
    layer.fused = not args.stepwise
    T_r = cfg.T // ep
    x = synth.tokens(cfg).cuda()[rank * T_r:(rank + 1) * T_r].contiguous()
    dy = synth.grad_output(cfg).cuda()[rank * T_r:(rank + 1) * T_r].contiguous()
    place = None
    state_ok = True
    if args.rebalance:
        layer.forward(x)
        loads = layer.observe_loads()
        # the paper's external scheduler (reading R20): libmoe's imbalance equals
        # the oracle's, a threshold above it keeps the placement, one below it migrates
        from oracle import migration as mig
        imb0 = mig.imbalance(loads.numpy(), list(range(cfg.E)), ep)
        state_ok &= abs(layer.imbalance() - imb0) < 1e-12
        keep = layer.maybe_rebalance(threshold=imb0 + 1.0)
        state_ok &= keep[1] == 0 and keep[2] == 0 and layer.placement == list(range(cfg.E))
        imb, swaps, moved = layer.maybe_rebalance(threshold=1.0)
        state_ok &= abs(imb - imb0) < 1e-12
        place = list(layer.placement)
        inv = [0] * cfg.E
        for e_, s_ in enumerate(place):
            inv[s_] = e_
        state_ok &= moved > 0
        for i, nm in enumerate(("master", "m", "v")):
            t = layer.state(nm)
            for el in range(E_l):
                state_ok &= bool(torch.equal(t[el], code(inv[rank * E_l + el]) * (i + 1)))
    outs = []
    for it in range(args.iters):  # epoch reuse: repeated calls must be bit-identical
        # alternate the NEXT-1 tile-granular dispatch -> GEMM1 launch with the separate
        # dispatch + GEMM1 (fused path): both must give the same bits
        layer.tile_overlap = layer.tile_overlap_bwd = it % 2 == 0
        y = layer.forward(x).clone()
        dx = layer.backward(dy).clone()
        outs.append((y, dx, layer.dw_gu.clone()))
    graph_ok = True
    if args.graph:
        # replays must match the eager step bit for bit (every replay is a fresh exchange), and
        # a replay on new input contents must match the eager step on those contents
        xg, dyg = x.clone(), dy.clone()
        yb, dxb, dwb = torch.empty_like(x), torch.empty_like(x), torch.empty_like(layer.dw_gu)

        def post():
            yb.copy_(layer.y)
            dxb.copy_(layer.dx)
            dwb.copy_(layer.dw_gu)
        graph = layer.capture(xg, dyg, post=post)
        for _ in range(args.iters):
            graph.replay()
            outs.append((yb.clone(), dxb.clone(), dwb.clone()))
        x2 = synth.tokens(cfg, seed=11).cuda()[rank * T_r:(rank + 1) * T_r].contiguous()
        xg.copy_(x2)
        graph.replay()
        y2g = yb.clone()
        y2e = layer.forward(x2).clone()
        layer.backward(dy)
        graph_ok = bool(torch.equal(y2g, y2e)) and not torch.equal(y2g, outs[0][0])
        layer.forward(x)     # the gathered layer state below is the step on x
        layer.backward(dy)
    torch.cuda.synchronize()
    st = layer.ctx.device_error()
    repeat_ok = all(torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1]) and
                    torch.equal(o[2], outs[0][2]) for o in outs[1:])
    y, dx, _ = outs[0]
    g = {
        "y": gather(y), "dx": gather(dx), "logits": gather(layer.logits),
        "topk": gather(layer.topk_idx), "dest": gather(layer.dest_row), "layout": gather(layer.layout),
        "dw_gu": gather(layer.dw_gu), "dw_down": gather(layer.dw_down), "dw_r": gather(layer.dw_r),
        "dgates": gather(layer.dgates),
    }
    if args.dedup:
        g["pdest"] = gather(layer.pdest)
        g["dlayout"] = gather(layer.dlayout)
        g["xr"] = gather(layer.xr)
    if cfg.E_s:
        g["dw_gu_s"] = gather(layer.dw_gu_s)
        g["dw_down_s"] = gather(layer.dw_down_s)
    flags = torch.tensor([st, int(repeat_ok and graph_ok and state_ok)], device="cuda")
    allflags = gather(flags)
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    if cfg.T == 0:
        zero = all(bool((t == 0).all()) for k in ("dw_gu", "dw_down", "dw_r", "dw_gu_s", "dw_down_s")
                   for t in g[k])
        lay0 = all(int(t.abs().sum()) == 0 for t in g["layout"])
        res = {"config": cfg.name, "ep": ep, "device_status": [int(f[0]) for f in allflags],
               "repeat_bitwise": [bool(f[1]) for f in allflags], "zero_grads": zero,
               "empty_layout": lay0}
        res["ok"] = (zero and lay0 and all(int(f[0]) == 0 for f in allflags) and
                     all(bool(f[1]) for f in allflags))
        print(json.dumps(res), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        return
    cat = lambda k: torch.cat(g[k]).cpu()
    x_all = synth.tokens(cfg)
    dy_all = synth.grad_output(cfg)
    logits = cat("logits").numpy()
    fw, bw = oracle_layer(cfg, x_all, dy_all, logits, ep=ep)
    res = {"config": cfg.name, "ep": ep, "rebalanced": place is not None, "device_status": [int(f[0]) for f in allflags],
           "repeat_bitwise": [bool(f[1]) for f in allflags]}
    checks = {}
    checks["topk"] = bool((cat("topk").numpy() == fw["topk_idx"]).all())
    checks["dest_row"] = all(bool((g["dest"][r].cpu().numpy() == fw["plan"]["ranks"][r]["dest_row"]).all())
                             for r in range(ep))
    E_l = cfg.E // ep
    lay_ok = True
    from oracle import moe_ref as ref
    padded = ref.recv_layout(fw["plan"]["counts_all"], ep, align=128, placement=place)
    for r in range(ep):
        lay = g["layout"][r].cpu().numpy()
        lay_ok &= bool((lay[:ep * cfg.E].reshape(ep, cfg.E) == fw["plan"]["counts_all"]).all())
        lay_ok &= bool((lay[ep * cfg.E:ep * cfg.E + E_l] == padded[r]["expert_rows"]).all())
        lay_ok &= bool((lay[ep * cfg.E + E_l:] == padded[r]["seg_base"]).all())
    checks["layout"] = lay_ok
    if args.dedup:
        from oracle import dedup as dd
        P = dd.plan(fw["topk_idx"], fw["gates"], cfg.E, ep, fw["C"], align=128, placement=place)
        ok = True
        for r in range(ep):
            pb = P["layout"]["pair_base"][r]
            ts = P["pairs"][r]["tslot"]
            want = np.where(ts >= 0, ts + pb[None, :], -1)
            ok &= bool((g["pdest"][r].cpu().numpy() == want).all())
            ok &= bool((g["dlayout"][r].cpu().numpy() == P["ntok_all"].reshape(-1)).all())
        checks["dedup_pairs"] = ok
        # every owner's expanded receive buffer holds x rows at the plain receive layout
        xa = x_all
        base = P["base"]   # receive rows under the placement in force (migration included)
        ok = True
        for q in range(ep):
            xr = g["xr"][q].cpu()
            t, j = np.nonzero((base["recv_row"] >= 0) & (base["owner"] == q))
            ok &= bool(torch.equal(xr[torch.as_tensor(base["recv_row"][t, j])], xa[torch.as_tensor(t)]))
        checks["dedup_xr"] = ok
    errs = {}
    errs["y"] = rel_err(f64(cat("y")), fw["y"])
    errs["dx"] = rel_err(f64(cat("dx")), bw["dx"])
    errs["dgates"] = rel_err(f64(cat("dgates")), bw["dgates"])
    errs["dW_r"] = rel_err(sum(f64(t) for t in g["dw_r"]).T, bw["dW_r"])
    errs["y_rows"] = rel_err_rows(f64(cat("y")), fw["y"])
    errs["dx_rows"] = rel_err_rows(f64(cat("dx")), bw["dx"])
    errs["dgates_rows"] = rel_err_rows(f64(cat("dgates")), bw["dgates"])
    f = cfg.f
    for e in range(cfg.E):
        q, el = divmod(e if place is None else place[e], E_l)
        if fw["cache"][e] is None:
            continue
        dgu = f64(g["dw_gu"][q][el])
        errs[f"dW_gate{e}"] = rel_err(dgu[:f].T, bw["dW_gate"][e])
        errs[f"dW_up{e}"] = rel_err(dgu[f:].T, bw["dW_up"][e])
        errs[f"dW_down{e}"] = rel_err(f64(g["dw_down"][q][el]).T, bw["dW_down"][e])
    if cfg.E_s:
        fs = cfg.E_s * cfg.f
        dgs = sum(f64(t[0]) for t in g["dw_gu_s"])     # per-rank partials sum to the global grad
        errs["dW_gate_s"] = rel_err(dgs[:fs].T, bw["dW_gate_s"])
        errs["dW_up_s"] = rel_err(dgs[fs:].T, bw["dW_up_s"])
        errs["dW_down_s"] = rel_err(sum(f64(t[0]) for t in g["dw_down_s"]).T, bw["dW_down_s"])
    worst = max(errs, key=errs.get)
    res.update(checks=checks, worst=[worst, errs[worst]], y=errs["y"], dx=errs["dx"])
    res["ok"] = (all(checks.values()) and all(v < TOL for v in errs.values()) and
                 all(s == 0 for s in res["device_status"]) and all(res["repeat_bitwise"]))
    if not res["ok"]:
        res["bad"] = {k: v for k, v in errs.items() if not v < TOL}
    print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

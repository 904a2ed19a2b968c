"""torchrun worker of the PP x EP pipelined executor (NEXT-3): every rank runs its stage's
layers in 1F1B order; rank 0 gathers every layer's inputs, outputs, logits and gradients and
checks each (layer, micro-batch) against the fp64 oracle teacher-forced with the GPU's own
inputs and logits, the stage-to-stage hand-offs bitwise, and the accumulated weight
gradients against the oracle's sum over micro-batches (tests/test_gpu_multi.py launches it).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tests/mp_pipe_worker.py --pp 2
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

CFG = synth.MoEConfig("pipe_small", T=512, d=256, E=8, k=2, f=256, cf=1.25)


gather = mp_common.gather


def layer_weights(g, experts, device):
    """Layer g's weights: the synth draws scaled per layer (so the layers differ)."""
    s = 1.0 + 0.125 * g
    w_gu, w_down = synth.expert_weights(CFG, experts, device=device)
    w_r = synth.router_weight(CFG, device=device)
    return ((w_r.float() * s).bfloat16(), (w_gu.float() * s).bfloat16(),
            (w_down.float() / s).bfloat16())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pp", type=int, default=2)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--micro", type=int, default=4)
    ap.add_argument("--dedup", default=None)
    ap.add_argument("--migrate", action="store_true",
                    help="after the warm-up step every stage migrates its layers' experts to a "
                         "seeded placement (PipelineStack.migrate: peer-store moves inside the "
                         "stage's EP subgroup)")
    ap.add_argument("--graph", action="store_true",
                    help="also replay the step from a CUDA graph: bitwise equal to eager")
    ap.add_argument("--tile", action="store_true",
                    help="force the tile-granular transfers (dispatch inside GEMM1, combine_bwd "
                         "inside dgrad-1) in every layer of the stack (NEXT-1 x NEXT-3)")
    args = ap.parse_args()
    local, shared = mp_common.init()
    world, rank = dist.get_world_size(), dist.get_rank()
    pp, M, Lyr = args.pp, args.micro, args.layers
    ep = world // pp
    stage, e = divmod(rank, ep)
    from paper_2605_05049_b200 import LayerDims
    from paper_2605_05049_b200.pipeline import PipelineStack
    from tests.helpers import TOL, f64, paper_weights, rel_err, rel_err_rows
    cfg = CFG
    T_r = cfg.T // ep
    dims = LayerDims(T_r, cfg.d, cfg.E, cfg.k, cfg.f, 0, cfg.cf, ep, e)
    stack = PipelineStack(dims, Lyr, pp, M, device=local, dedup=args.dedup)
    if args.tile:
        for slots in stack.layers:
            for s_ in slots:
                s_.tile_overlap = s_.tile_overlap_bwd = True
    E_l = cfg.E // ep
    dev = torch.device(f"cuda:{local}")
    per = Lyr // pp
    for l in range(per):
        w_r, w_gu, w_down = layer_weights(stage * per + l, range(e * E_l, (e + 1) * E_l), dev)
        stack.set_weights(l, w_r, w_gu, w_down)
    x_all = synth.tokens(cfg, T=M * cfg.T).cuda().view(M, cfg.T, cfg.d)
    dy_all = synth.grad_output(cfg, T=M * cfg.T).cuda().view(M, cfg.T, cfg.d)
    xs = [x_all[m, e * T_r:(e + 1) * T_r].contiguous() for m in range(M)]
    dys = [dy_all[m, e * T_r:(e + 1) * T_r].contiguous() for m in range(M)]
    stack.step(xs if stage == 0 else None, dys if stage == pp - 1 else None)   # warm-up step
    place_of = lambda s_: (list(np.random.default_rng(100 + s_).permutation(cfg.E))
                           if args.migrate else list(range(cfg.E)))
    moved = 0
    if args.migrate:
        for l in range(per):
            moved += stack.migrate(l, place_of(stage))
    graph_ok = True
    if args.graph:
        a_in, a_dy = (xs if stage == 0 else None), (dys if stage == pp - 1 else None)
        ye, dxe = stack.step(a_in, a_dy)
        ye = [t.clone() for t in ye] if ye is not None else None
        dxe = [t.clone() for t in dxe] if dxe is not None else None
        dwe = [t.clone() for t in stack.grads(0)]
        graph = stack.capture(a_in, a_dy)
        graph.replay()
        torch.cuda.synchronize()
        if ye is not None:
            graph_ok &= all(torch.equal(u, v) for u, v in zip(ye, stack.y_out))
        if dxe is not None:
            graph_ok &= all(torch.equal(u, v) for u, v in zip(dxe, stack.dx_out))
        graph_ok &= all(torch.equal(u, v) for u, v in zip(dwe, stack.grads(0)))
        del graph
    stack.record = {}
    ys, dxs = stack.step(xs if stage == 0 else None, dys if stage == pp - 1 else None)
    torch.cuda.synchronize()
    status = max(s.ctx.device_error() for slots in stack.layers for s in slots)
    rec = stack.record
    # the stack's local layer 0 against a plain MoELayer with the same weights on the same
    # recorded input and upstream gradient: y, dx and (M = 1) the weight gradients bitwise
    from paper_2605_05049_b200 import MoELayer
    plain = MoELayer(dims, device=local, group=stack.group, dedup=args.dedup)
    w_r, w_gu, w_down = layer_weights(stage * per, range(e * E_l, (e + 1) * E_l), dev)
    plain.set_weights(w_r, w_gu, w_down)
    if args.migrate:
        plain.migrate(place_of(stage))
    yp = plain.forward(rec[(0, 0)]["x"]).clone()
    dxp = plain.backward(rec[(0, 0)]["dy"]).clone()
    torch.cuda.synchronize()
    dflag = [torch.equal(yp, rec[(0, 0)]["y"]), torch.equal(dxp, rec[(0, 0)]["dx"])]
    if M == 1:
        dflag += [torch.equal(plain.dw_gu, stack.grads(0)[1]),
                  torch.equal(plain.dw_down, stack.grads(0)[2]),
                  torch.equal(plain.dw_r, stack.grads(0)[0])]
    direct = all(dflag)
    plain.close()
    # PAPER.md Eq. 4 per-stage memory account (measured bytes of every activation context)
    mem_all = [None] * world
    dist.all_gather_object(mem_all, stack.memory_report())
    # gather: [rank][local layer][m] tensors
    keys = ["x", "y", "logits", "topk", "dest", "dy", "dx"]
    G = {k: [[gather(rec[(l, m)][k]) for m in range(M)] for l in range(per)] for k in keys}
    dW = [[gather(t) for t in stack.grads(l)] for l in range(per)]   # dw_r, dw_gu, dw_down
    st = gather(torch.tensor([status], device=dev))
    dflags = gather(torch.tensor([int(direct)], device=dev))
    gflags = gather(torch.tensor([int(graph_ok)], device=dev))
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    from oracle import moe_ref as ref
    from tests.helpers import ALIGN
    local_path = ep == 1 and stack.layers[0][0].local_fast_path and not stack.layers[0][0].dedup
    errs, checks = {}, {"routing": True, "handoff": True}
    errs_norm = {}
    ranks_of = lambda s_: list(range(s_ * ep, (s_ + 1) * ep))
    for g in range(Lyr):
        s_, l = divmod(g, per)
        rs = ranks_of(s_)
        W = layer_weights(g, range(cfg.E), "cuda")
        w_r = f64(W[0]).T
        Wg, Wu, Wd = zip(*[paper_weights(W[1][x], W[2][x], cfg.f) for x in range(cfg.E)])
        dWg = dWu = dWd = dWr = None
        for m in range(M):
            cat = lambda k: torch.cat([G[k][l][m][r] for r in rs]).cpu()
            X, Y, LG, DY, DX = cat("x"), cat("y"), cat("logits"), cat("dy"), cat("dx")
            fw, bw = ref.layer_forward_backward(f64(X), w_r, Wg, Wu, Wd, f64(DY), cfg.k, cfg.cf,
                                                ep, logits=LG.numpy())
            checks["routing"] &= bool((cat("topk").numpy() == fw["topk_idx"]).all())
            if local_path:   # EP = 1 receive-layout path: dest_row = 128-aligned receive row
                want = [ref.dispatch_plan(fw["topk_idx"], cfg.E, 1, fw["C"], align=ALIGN)["recv_row"]]
            else:
                want = [fw["plan"]["ranks"][i]["dest_row"] for i in range(len(rs))]
            for i, r in enumerate(rs):
                checks["routing"] &= bool((G["dest"][l][m][r].cpu().numpy() == want[i]).all())
            errs[f"y{g}.{m}"] = rel_err(f64(Y), fw["y"])
            errs[f"dx{g}.{m}"] = rel_err(f64(DX), bw["dx"])
            errs[f"y_rows{g}.{m}"] = rel_err_rows(f64(Y), fw["y"])
            errs[f"dx_rows{g}.{m}"] = rel_err_rows(f64(DX), bw["dx"])
            acc = lambda a, b: b if a is None else [u + v for u, v in zip(a, b)]
            dWg, dWu, dWd = acc(dWg, bw["dW_gate"]), acc(dWu, bw["dW_up"]), acc(dWd, bw["dW_down"])
            dWr = bw["dW_r"] if dWr is None else dWr + bw["dW_r"]
            # hand-offs: layer g's output is layer g+1's input, layer g+1's dx is layer g's dy
            if g + 1 < Lyr:
                s2, l2 = divmod(g + 1, per)
                for i in range(ep):
                    r1, r2 = rs[i], ranks_of(s2)[i]
                    checks["handoff"] &= bool(torch.equal(G["y"][l][m][r1], G["x"][l2][m][r2]))
                    checks["handoff"] &= bool(torch.equal(G["dy"][l][m][r1], G["dx"][l2][m][r2]))
        for x in range(cfg.E):
            q, el = divmod(int(place_of(s_)[x]), E_l)
            r = rs[q]
            dgu = f64(dW[l][1][r][el])
            errs[f"dWg{g}.{x}"] = rel_err(dgu[:cfg.f].T, dWg[x])
            errs[f"dWu{g}.{x}"] = rel_err(dgu[cfg.f:].T, dWu[x])
            errs[f"dWd{g}.{x}"] = rel_err(f64(dW[l][2][r][el]).T, dWd[x])
            if x == 0:
                errs_norm[f"dWd{g}.0"] = float(np.linalg.norm(f64(dW[l][2][r][el]).T) /
                                               max(np.linalg.norm(dWd[x]), 1e-30))
        errs[f"dWr{g}"] = rel_err(sum(f64(dW[l][0][r]) for r in rs).T, dWr)
    # Eq. 4: stage i keeps PP - i in-flight micro-batches (min with M); the measured memory
    # difference between the first and last stage is exactly (PP - 1) L/PP activation contexts
    # (PAPER.md:334-341 Delta M); each context saves 2 R (3f + d) bytes of expert activations
    # for R = recv_rows_max >= Eq. 4's 2 T_local k (3f + d) (the capacity / alignment slack)
    mem_ok = True
    for mr in mem_all:
        mem_ok &= all(l["n_slots"] == mr["in_flight_bound"] for l in mr["layers"])
        mem_ok &= mr["in_flight_bound"] == min(pp - mr["stage"], M)
        for l in mr["layers"]:
            mem_ok &= all(v >= mr["eq4_expert_activation_bytes_per_microbatch"]
                          for v in l["saved_expert_activation_bytes"])
    first = [mr for mr in mem_all if mr["stage"] == 0]
    last = [mr for mr in mem_all if mr["stage"] == pp - 1]
    slot_b = first[0]["layers"][0]["slot_total_bytes"][-1]       # a non-owner context
    dM = first[0]["stage_bytes"] - last[0]["stage_bytes"]
    if pp > 1 and M >= pp:
        mem_ok &= dM == (pp - 1) * per * slot_b
    eq4 = first[0]["eq4_expert_activation_bytes_per_microbatch"]
    checks["eq4_memory"] = bool(mem_ok)
    res_mem = {"stage_bytes": [mr["stage_bytes"] for mr in mem_all],
               "delta_M_measured": dM, "delta_M_eq4_expert_term": (pp - 1) * per * eq4,
               "context_bytes": slot_b,
               "saved_over_eq4": first[0]["layers"][0]["saved_expert_activation_bytes"][0] / eq4}
    worst = max(errs, key=errs.get)
    checks["direct_layer0"] = all(bool(t.item()) for t in dflags)
    checks["graph_replay"] = all(bool(t.item()) for t in gflags)
    res = {"pp": pp, "ep": ep, "migrated": bool(args.migrate), "layers": Lyr, "micro": M, "checks": checks,
           "device_status": [int(t.item()) for t in st], "worst": [worst, errs[worst]],
           "schedule_stage0": stack.ops if stage == 0 else None, "memory": res_mem}
    res["ok"] = (all(checks.values()) and all(v < TOL for v in errs.values()) and
                 all(v == 0 for v in res["device_status"]))
    if not res["ok"]:
        res["bad"] = {k: v for k, v in errs.items() if not v < TOL}
        res["norm_ratio"] = errs_norm
    print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

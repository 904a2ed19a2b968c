"""Benchmark of the expert-parallel MoE layer fwd+bwd (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mixtral|dsmoe|dsv3|tiny]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference ...   # the fp64 CPU oracle (the only reference this tier has)
    python bench.py --a2a                  # dispatch/combine GB/s sweep vs NCCL all_to_all
    python bench.py --config dsmoe|dsv3 [--rebalance] [--dedup [dispatch|all]]  # fine-grained
    torchrun ... bench.py --gpus 4 --pp 2 [--graph]   # NEXT-3 PP x EP 1F1B stack (own metric)

A "step" is one forward + backward of the whole layer
over T tokens of the EP group (T/N per rank, experts sharded E/N per rank).  At N=1 the
workload is the Mixtral-8x7B layer (BASELINE.json configs[1]: d=4096 E=8 top-2 f=14336
T=8192, cf=1.25); N>1 shards the same T=8192 tokens (strong scaling).  Timing: CUDA
events on the launching stream, barrier + synchronize on both sides, max over ranks.
Inputs (the 2.8 GB of bf16 expert weights per GPU at N=1) are larger than L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "MoE layer fwd+bwd tokens/s"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="mixtral", choices=list(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--a2a", action="store_true", help="dispatch/combine sweep vs NCCL")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rebalance", action="store_true",
                    help="expert migration before timing: observe loads, Alg. 2, move experts")
    ap.add_argument("--dedup", nargs="?", const="dispatch", default=None,
                    choices=["dispatch", "all"],
                    help="NEXT-4 deduplicated all-to-alls (one row per (token, owner) pair): "
                         "'dispatch' = dispatch + combine_bwd (default), 'all' = all four")
    ap.add_argument("--stepwise", action="store_true",
                    help="step-by-step C-ABI calls instead of the fused compute+all-to-all ones")
    ap.add_argument("--cpu-sample-tokens", type=int, default=0)
    ap.add_argument("--breakdown", action="store_true",
                    help="per-phase CUDA-event breakdown of a step (max over ranks), no bench line")
    ap.add_argument("--comm-sms", type=int, default=None,
                    help="SMs given to an all-to-all running beside a GEMM (MoELayer.comm_sms)")
    ap.add_argument("--graph", action="store_true",
                    help="also time the step replayed from a CUDA graph (MoELayer.capture); "
                         "the headline uses the faster of eager / graph")
    ap.add_argument("--gemm-compare", action="store_true",
                    help="expert FFN GEMMs: libmoe vs cuBLAS (torch) on one GPU, no bench line")
    ap.add_argument("--gemm-experts", type=int, default=0,
                    help="--gemm-compare: experts on the GPU (default: the config's E)")
    ap.add_argument("--gemm-rows", type=int, default=0,
                    help="--gemm-compare: rows per expert (default: T*k/E)")
    ap.add_argument("--pp", type=int, default=1,
                    help="NEXT-3: PP x EP pipelined stack (world = PP x EP), 1F1B over --micro")
    ap.add_argument("--layers", type=int, default=4, help="--pp: MoE layers in the stack")
    ap.add_argument("--micro", type=int, default=8, help="--pp: micro-batches per step")
    ap.add_argument("--migrate-bench", action="store_true",
                    help="NEXT-2: time moe_migrate moving every expert's full training state "
                         "(bf16 weights, fp32 grads, fp32 master + Adam moments) to another "
                         "rank, against PAPER.md's 48 d f bytes per expert at 50 GB/s")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="run only this many steps without timing (for ncu)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local, backend="nccl"):
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend, device_id=torch.device(f"cuda:{local}")
                                if backend == "nccl" else None)
        return dist
    return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            m = json.load(fh)
        return dict(hbm=m.get("hbm_gbs", 6650.0), bf16=m.get("bf16_tflops", 1590.0),
                    bf16_sustained=m.get("bf16_tflops_sustained", 1400.0), source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, source="fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"moe_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
            return
        # nvidia-smi needs ~0.1-0.3 s to print its first line: wait for it, so that a short
        # timed region (a few ms per step) still has samples taken under its load
        t0 = time.time()
        while time.time() - t0 < 3.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.01)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def gemm_traffic(config, world):
    """DRAM bytes per step of the 6 expert-GEMM launches from the committed ncu --set full
    capture (profiles/gemm_traffic.json), for the configuration it was captured on."""
    p = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    key = f"{config}_ep{world}"
    try:
        with open(p) as fh:
            return json.load(fh)[key]["dram_bytes_per_step"]
    except (OSError, KeyError, ValueError):
        return None


def gemm_ncu(config, world):
    """Per-launch ncu metrics of the 6 expert-GEMM launches (tensor-pipe %, SM clock, DRAM
    bytes) from the committed --set full capture (profiles/gemm_ncu.json), if captured for
    this configuration."""
    p = os.path.join(ROOT, "profiles", "gemm_ncu.json")
    try:
        with open(p) as fh:
            return json.load(fh)[f"{config}_ep{world}"]
    except (OSError, KeyError, ValueError):
        return None


def layer_roofline(layer, cfg, peaks, nvl_gbs=900.0, sustained=False):
    """SURVEY.md §8(d) d.3 serial layer roofline from the realised routing (the layout
    record's [EP x E] count matrix and the expert placement, identical on every rank):
    sum over the steps of max(F/pi, B_hbm/beta_hbm, B_nvl/beta_nvl) on the hottest rank,
    pi = measured bf16 (burst; sustained=True: the 4 s back-to-back figure),
    beta_hbm = measured HBM copy bandwidth, beta_nvl = 900 GB/s
    per direction.  Steps: router GEMM (fwd + 2 bwd), permute / unpermute / permute_bwd /
    combine_bwd's dO writes (HBM), 4 all-to-alls (NVLink, max of egress and ingress), expert
    GEMMs fwd + bwd (18 d f per routed row, shared experts on the local tokens)."""
    EP, E, d, f, k = layer.dims.ep_size, cfg.E, cfg.d, cfg.f, cfg.k
    T_r = layer.dims.T_local
    cm = layer.layout[:EP * E].view(EP, E).to(torch.int64).cpu()
    owner = torch.tensor([s // layer.E_l for s in layer.placement])
    pi_tf = peaks["bf16_sustained"] if sustained else peaks["bf16"]
    pi = pi_tf * 1e12
    bh = peaks["hbm"] * 1e9
    bn = nvl_gbs * 1e9
    row = d * 2
    per_rank = []
    for r in range(EP):
        mine = owner == r
        recv = int(cm[:, mine].sum())
        send = int(cm[r].sum())
        egress = int(cm[r, ~mine].sum()) * row
        ingress = int(cm[:, mine].sum() - cm[r, mine].sum()) * row
        t = 3 * 2 * T_r * d * E / pi                          # router fwd + dgrad + wgrad
        if layer.dedup:
            # pairs instead of slots on NVLink in the deduplicated directions; HBM: the owner's
            # expands (pairs -> receive rows), and for mode "all" the pair reduces / gathers
            nm = layer.dlayout.view(EP, EP).to(torch.int64).cpu()
            pairs_out, pairs_in = int(nm[r].sum()), int(nm[:, r].sum())
            p_egress = (pairs_out - int(nm[r, r])) * row
            p_ingress = (pairs_in - int(nm[r, r])) * row
            t += 2 * (pairs_in * row + recv * row) / bh         # fwd expand, bwd expand (dO)
            if layer.dedup_mode == "all":
                t += 2 * (pairs_out * row + T_r * row) / bh     # y / dx gathers over pairs
                t += 2 * (recv * row + pairs_in * row) / bh     # combine / dispatch_bwd reduces
                t += recv * row / bh                            # bwd expand reads O for dg
                t += 4 * max(p_egress, p_ingress) / bn
            else:
                t += (T_r * row + send * row) / bh              # dgates dots at the source
                t += 2 * (send * row + T_r * row) / bh          # unpermute, permute_bwd
                t += 2 * max(p_egress, p_ingress) / bn + 2 * max(egress, ingress) / bn
        else:
            t += 2 * (T_r * row + send * row) / bh            # permute, permute_bwd
            t += 2 * (send * row + T_r * row) / bh            # unpermute, combine_bwd dO rows
            t += 4 * max(egress, ingress) / bn                # dispatch, combine, their twins
        t += 18 * recv * d * f / pi                           # expert GEMMs fwd + bwd
        if cfg.E_s:
            t += 18 * T_r * d * cfg.E_s * f / pi
        per_rank.append(t * 1e3)
    hot = max(range(EP), key=lambda r: per_rank[r])
    return {"serial_ms": per_rank[hot], "hot_rank": hot,
            "per_rank_ms": [round(v, 4) for v in per_rank],
            "peaks": {"bf16_tflops": pi_tf, "hbm_gbs": peaks["hbm"],
                      "nvlink_gbs_per_direction": nvl_gbs}}


def realised_gemm_flops(layer, cfg):
    """Algorithmic GEMM FLOPs of one fwd+bwd on this rank from the realised routing:
    6 * rows * d * f (fwd) + 12 * rows * d * f (bwd), plus the shared experts."""
    rows = int(layer.expert_rows.sum().item())
    fl = 18 * rows * cfg.d * cfg.f
    if cfg.E_s:
        fl += 18 * layer.dims.T_local * cfg.d * cfg.E_s * cfg.f
    return fl


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    world, rank, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    from paper_2605_05049_b200 import LayerDims, MoELayer

    cfg = synth.CONFIGS[args.config]
    ep = world
    T_r = cfg.T // ep
    dims = LayerDims(T_r, cfg.d, cfg.E, cfg.k, cfg.f, cfg.E_s, cfg.cf, ep, rank)
    layer = MoELayer(dims, device=local, fused=not args.stepwise, dedup=args.dedup)
    if os.environ.get("MOE_EP1_GENERAL") == "1":   # measurements: EP = 1 through permute + dispatch
        layer.local_fast_path = False
    if args.comm_sms is not None:
        layer.comm_sms = args.comm_sms
    E_l = cfg.E // ep
    dev = torch.device(f"cuda:{local}")
    w_gu, w_down = synth.expert_weights(cfg, range(rank * E_l, (rank + 1) * E_l), device=dev)
    w_gu_s, w_down_s = synth.shared_weights(cfg, device=dev)
    layer.set_weights(synth.router_weight(cfg, device=dev), w_gu, w_down, synth.zipf_bias(cfg),
                      w_gu_s, w_down_s)
    x_all = synth.tokens(cfg, device=dev)
    dy_all = synth.grad_output(cfg, device=dev)
    x = x_all[rank * T_r:(rank + 1) * T_r].contiguous()
    dy = dy_all[rank * T_r:(rank + 1) * T_r].contiguous()
    del x_all, dy_all
    stream = torch.cuda.current_stream()

    def breakdown():
        """Per-phase CUDA-event times of a step (ranks barrier-aligned before every step, so
        a phase that waits for a peer shows load imbalance, not launch skew)."""
        acc = {}
        for _ in range(args.steps):
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            layer.marks = []
            layer.forward(x)
            layer.backward(dy)
            torch.cuda.synchronize()
            prev = layer.marks[0][1]
            for name, ev in layer.marks[1:]:
                acc[name] = acc.get(name, 0.0) + prev.elapsed_time(ev)
                prev = ev
        layer.marks = None
        names = list(acc)
        v = torch.tensor([acc[n] / args.steps for n in names], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
        if rank == 0:
            tot = sum(v.tolist())
            print(json.dumps({"breakdown_ms_max_over_ranks": {n: round(t, 4) for n, t in zip(names, v.tolist())},
                              "sum_ms": tot, "config": args.config, "n_gpus": world,
                              "rebalanced": bool(args.rebalance)}))
        layer.close()
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()

    if args.profile_steps:
        for _ in range(args.profile_steps):
            layer.forward(x)
            layer.backward(dy)
        torch.cuda.synchronize()
        layer.ctx.check_device_error()
        if rank == 0:
            print(json.dumps({"profile_steps": args.profile_steps, "config": args.config}))
        return

    def barrier():
        if dist is not None:
            dist.barrier()

    # Region events inside the timed steps, on the stream each call is issued on: the
    # grouped-GEMM family (the dominant kernel: 6 launches per step), the permute (HBM) and
    # the two forward-pattern all-to-alls (NVLink)
    gemm_ev = []
    region_ev = {"permute": [], "dispatch": [], "combine_bwd": []}
    import paper_2605_05049_b200.layer as layer_mod

    def timed(fn, bucket=None):
        def wrapper(*a, **kw):
            st = kw.get("stream") or stream
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            fn(*a, **kw)
            e.record(st)
            (gemm_ev if bucket is None else region_ev[bucket]).append((s, e))
        return wrapper

    for _ in range(args.warmup):
        layer.forward(x)
        layer.backward(dy)
    torch.cuda.synchronize()
    layer.ctx.check_device_error()
    rebal = None
    if args.rebalance:
        # expert migration (§VI): observe the routed load per expert, run Alg. 2,
        # move the experts, re-warm; the migration itself is outside the timed steps
        def rank_rows():
            n = torch.tensor([int(layer.expert_rows.sum().item())], device=dev)
            if dist is not None:
                allr = [torch.zeros_like(n) for _ in range(world)]
                dist.all_gather(allr, n)
                return [int(v.item()) for v in allr]
            return [int(n.item())]
        before = rank_rows()
        for _ in range(3):
            layer.forward(x)
            layer.observe_loads()
            layer.backward(dy)
        swaps, moved = layer.rebalance()
        for _ in range(args.warmup):
            layer.forward(x)
            layer.backward(dy)
        torch.cuda.synchronize()
        rebal = {"swaps": swaps, "experts_moved": moved, "rank_rows_before": before,
                 "rank_rows_after": rank_rows()}
    if args.breakdown:
        return breakdown()

    # ---- device-timed region: the plain step loop, nothing else on the stream (`value`)
    clocks = ClockSampler(local)
    # the sampler first (it waits up to ~0.3 s for nvidia-smi's first line, a different time
    # on every rank), THEN the barrier: the ranks enter the timed loop together
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        layer.forward(x)
        layer.backward(dy)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    layer.ctx.check_device_error()
    ms = t0.elapsed_time(t1) / args.steps
    eager_ms = ms
    graph_ms = None
    if args.graph:
        # the same step replayed from one CUDA graph (no host launch overhead)
        graph = layer.capture(x, dy)
        for _ in range(args.warmup):
            graph.replay()
        clocks.start()
        barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        clk_g = clocks.stop()
        layer.ctx.check_device_error()
        graph_ms = t0.elapsed_time(t1) / args.steps
        del graph

    # ---- a SEPARATE instrumented pass for the per-kernel regions (roofline.achieved): CUDA
    # events around the C-ABI calls, on the stream each call is issued on -- the grouped-GEMM
    # family (the dominant kernel: 6 launches per step), the permute (HBM) and the two
    # forward-pattern all-to-alls (NVLink).  Not part of `value`.
    hooked = ["moe_expert_ffn", "moe_expert_ffn_bwd", "moe_expert_ffn_combine",
              "moe_expert_ffn_bwd_dispatch", "moe_expert_ffn_up", "moe_expert_ffn_down_combine",
              "moe_expert_ffn_bwd_dh", "moe_expert_ffn_bwd_dx_dispatch",
              # GEMM1 / dgrad-1 launches that carry the dispatch / combine_bwd (NEXT-1): their
              # time counts as GEMM time, the transfer regions then stay empty
              "moe_dispatch_expert_ffn_up", "moe_combine_bwd_expert_ffn_dh"]
    buckets = {"moe_permute": "permute", "moe_permute_dispatch_local": "permute",
               "moe_dispatch": "dispatch",
               "moe_combine_bwd": "combine_bwd", "moe_combine_bwd_local": "combine_bwd",
               "moe_dedup_dispatch": "dispatch",
               "moe_dedup_combine_bwd": "combine_bwd", "moe_dedup_combine_bwd_ys": "combine_bwd"}
    originals = {n: getattr(layer_mod.L, n) for n in hooked + list(buckets)}
    for n in hooked:
        setattr(layer_mod.L, n, timed(originals[n]))
    for n, b in buckets.items():
        setattr(layer_mod.L, n, timed(originals[n], b))
    barrier()
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(args.steps):
        layer.forward(x)
        layer.backward(dy)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    for n, fn in originals.items():
        setattr(layer_mod.L, n, fn)
    layer.ctx.check_device_error()
    instr_ms = t0.elapsed_time(t1) / args.steps
    region_ms = {b: sum(a.elapsed_time(z) for a, z in ev) / args.steps
                 for b, ev in region_ev.items()}
    gemm_ms = sum(s.elapsed_time(e) for s, e in gemm_ev) / args.steps
    gemm_flops = realised_gemm_flops(layer, cfg)

    # ---- end-to-end through the public API with host buffers (pinned), copies timed
    x_h = x.cpu().pin_memory()
    dy_h = dy.cpu().pin_memory()
    y_h = torch.empty_like(x_h).pin_memory()
    dx_h = torch.empty_like(x_h).pin_memory()
    # Pipelined: every step's inputs go host->device and its outputs device->host on a copy
    # stream (PCIe both directions), overlapping the neighbouring steps' compute; all copies
    # of all K steps are inside the timed region (first H2D .. last D2H).
    cs = torch.cuda.Stream(device=dev)
    x_d = [torch.empty_like(x) for _ in range(2)]
    dy_d = [torch.empty_like(dy) for _ in range(2)]
    y_b = [torch.empty_like(x) for _ in range(2)]
    dx_b = [torch.empty_like(x) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    with torch.cuda.stream(cs):
        x_d[0].copy_(x_h, non_blocking=True)
        dy_d[0].copy_(dy_h, non_blocking=True)
        ev_in[0].record(cs)
    for i in range(args.steps):
        s = i % 2
        stream.wait_event(ev_in[s])
        if i + 1 < args.steps:           # next step's inputs, once step i-1 released the slot
            with torch.cuda.stream(cs):
                if i >= 1:
                    cs.wait_event(ev_done[1 - s])
                x_d[1 - s].copy_(x_h, non_blocking=True)
                dy_d[1 - s].copy_(dy_h, non_blocking=True)
                ev_in[1 - s].record(cs)
        if i >= 2:
            stream.wait_event(ev_out[s])  # D2H of step i-2 finished reading y_b[s], dx_b[s]
        y = layer.forward(x_d[s])
        dxo = layer.backward(dy_d[s])
        y_b[s].copy_(y, non_blocking=True)
        dx_b[s].copy_(dxo, non_blocking=True)
        ev_done[s].record(stream)
        with torch.cuda.stream(cs):
            cs.wait_event(ev_done[s])
            y_h.copy_(y_b[s], non_blocking=True)
            dx_h.copy_(dx_b[s], non_blocking=True)
            ev_out[s].record(cs)
    e1.record(cs)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps

    # byte counts of this rank's permute and forward-pattern all-to-alls (realised routing)
    EPw, Ew, row_b = world, cfg.E, cfg.d * 2
    cmat = layer.layout[:EPw * Ew].view(EPw, Ew).to(torch.int64).cpu()
    own = torch.tensor([sl // layer.E_l for sl in layer.placement]) == rank
    send_rows = int(cmat[rank].sum())
    a2a_bytes = {"egress": int(cmat[rank, ~own].sum()) * row_b,
                 "ingress": int(cmat[:, own].sum() - cmat[rank, own].sum()) * row_b}
    permute_bytes = T_r * row_b + send_rows * row_b
    if layer.dedup:   # one row per (token, owner) pair; the permute moves indices only
        nm = layer.dlayout.view(EPw, EPw).to(torch.int64).cpu()
        a2a_bytes = {"egress": int(nm[rank].sum() - nm[rank, rank]) * row_b,
                     "ingress": int(nm[:, rank].sum() - nm[rank, rank]) * row_b}
        permute_bytes = T_r * cfg.k * 8
    roof = layer_roofline(layer, cfg, measured_peaks())
    roof_sus = layer_roofline(layer, cfg, measured_peaks(), sustained=True)
    vals = torch.tensor([ms, e2e_ms, gemm_ms, graph_ms or 0.0, region_ms["permute"], instr_ms],
                        dtype=torch.float64, device=dev)
    # a collective's kernel time on a rank includes waiting for the later ranks; the rank that
    # arrives last waits least, so the MIN over ranks is the transfer's own duration
    a2a_t = torch.tensor([region_ms["dispatch"], region_ms["combine_bwd"]], dtype=torch.float64,
                         device=dev)
    if dist is not None:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(a2a_t, op=dist.ReduceOp.MIN)
    ms, e2e_ms, gemm_ms_max, graph_ms, perm_ms, instr_ms = vals.tolist()
    disp_ms, cbwd_ms = a2a_t.tolist()
    eager_ms = ms
    use_graph = bool(args.graph and graph_ms < ms)
    if use_graph:
        ms = graph_ms
        clk = clk_g
    if rank != 0:
        layer.close()
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    tokens = cfg.T
    peaks = measured_peaks()
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12
    out = {
        "metric": METRIC,
        "value": tokens / (ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) tokens, random-init expert/router weights)",
        "config": {
            "workload": f"{cfg.name} MoE layer fwd+bwd",
            "T": cfg.T, "d": cfg.d, "E": cfg.E, "k": cfg.k, "f": cfg.f, "E_shared": cfg.E_s,
            "capacity_factor": cfg.cf, "zipf_s": cfg.zipf_s,
            "parallelism": f"ep{world}", "tokens_per_rank": T_r,
            "expert_migration": rebal,
            "dedup_a2a": layer.dedup_mode,
            # NEXT-1 tile-granular transfers (dispatch inside GEMM1 / combine_bwd inside
            # dgrad-1); only on the EP > 1 path
            "tile_overlap": {"fwd": world > 1 and layer._tile_overlap(),
                             "bwd": world > 1 and layer._tile_overlap_bwd()},
            "cuda_graph": use_graph,
            "eager_ms_per_step": eager_ms,
            "graph_ms_per_step": graph_ms if args.graph else None,
            "l2": "inputs larger than L2 (bf16 expert weights %.2f GB per GPU)" % (
                (w_gu.numel() + w_down.numel()) * 2 / 1e9),
        },
        "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": int(x_h.numel() * 2 + dy_h.numel() * 2),
                "d2h_bytes_per_step": int(y_h.numel() * 2 + dx_h.numel() * 2)},
        "layer_roofline": {
            **roof, "frac": roof["serial_ms"] / ms,
            "serial_ms_sustained_peak": roof_sus["serial_ms"],
            "frac_sustained_peak": roof_sus["serial_ms"] / ms,
            "definition": "SURVEY.md 8(d) d.3: sum over steps of max(F/pi, B_hbm/beta_hbm, "
                          "B_nvl/beta_nvl) on the hottest rank, realised routing; pi = measured "
                          "burst bf16 (frac), measured sustained bf16 (frac_sustained_peak)",
        },
        "secondary_rooflines": {
            "permute": {"bound": "hbm", "ms": perm_ms,
                        "achieved_gbs": permute_bytes / (perm_ms * 1e-3) / 1e9 if perm_ms else None,
                        "peak_gbs": peaks["hbm"], "bytes_rank0": permute_bytes,
                        "note": ("indices only (dedup: no xs scatter; the dedup dispatch reads x)"
                                 if layer.dedup else
                                 "3 kernels (histogram+scan, rank, scatter); algorithmic bytes = "
                                 "x read + xs write")},
            "dispatch": {"bound": "nvlink" if world > 1 else "hbm (EP=1: local copy)",
                         "ms": disp_ms, "egress_bytes_rank0": a2a_bytes["egress"],
                         "ingress_bytes_rank0": a2a_bytes["ingress"],
                         "achieved_gbs_per_direction": max(a2a_bytes.values()) / (disp_ms * 1e-3) / 1e9
                         if disp_ms and world > 1 else None,
                         "peak_gbs_per_direction": 900.0,
                         "note": "one launch incl. the counts handshake and padding zeroing; "
                                 "min over ranks of the in-step kernel time"},
            "combine_bwd": {"ms": cbwd_ms,
                            "achieved_gbs_per_direction": max(a2a_bytes.values()) / (cbwd_ms * 1e-3) / 1e9
                            if cbwd_ms and world > 1 else None,
                            "note": "forward pattern + gate multiply + dgates dot products"},
        },
        "gpu_launches": layer.kernel_launches() * args.steps,
        "clocks": clk,
        "roofline": {
            "kernel": "grouped_gemm_kernel (tcgen05 cta_group::2; 6 launches/step: GEMM1+SwiGLU, "
                      "GEMM2(+combine stores), dgrad-1+dSwiGLU, dgrad-2(+dispatch_bwd stores), "
                      "wgrad x2); timed region = the FFN C-ABI calls",
            "bound": "tensor",
            "achieved": achieved,
            "peak": peaks["bf16"],
            "unit": "TFLOP/s",
            "frac": achieved / peaks["bf16"],
            "peak_sustained": peaks["bf16_sustained"],
            "frac_sustained": achieved / peaks["bf16_sustained"],
            "traffic": gemm_traffic(args.config, world),
            "ncu": gemm_ncu(args.config, world),
            "peak_source": peaks["source"] + " bf16_tflops (burst, SURVEY.md 8(d) d.3); "
                           "frac_sustained against bf16_tflops_sustained",
            "algorithmic_flops_per_step": gemm_flops,
            "gemm_ms_per_step": gemm_ms,
            "gemm_share_of_step": gemm_ms / instr_ms,
            "timing": "achieved = FLOPs / the GEMM calls' CUDA-event time in a separate "
                      "instrumented pass (%.3f ms/step); value comes from the plain loop" % instr_ms,
        },
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_sample_tokens or 128, w_gu, w_down, layer)
    print(json.dumps(out), flush=True)
    layer.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- oracle arm
def _oracle_inputs(cfg, n_tok, w_gu=None, w_down=None):
    """Oracle inputs for a bounded sample: the first n_tok tokens of the workload and all
    E experts' weights as float32 (exact for bf16; the oracle computes in fp64)."""
    if w_gu is None:
        w_gu, w_down = synth.expert_weights(cfg, range(cfg.E))
    f = cfg.f
    Wg = [w_gu[e, :f].float().cpu().numpy().T for e in range(cfg.E)]
    Wu = [w_gu[e, f:].float().cpu().numpy().T for e in range(cfg.E)]
    Wd = [w_down[e].float().cpu().numpy().T for e in range(cfg.E)]
    x = synth.tokens(cfg, T=cfg.T)[:n_tok].float().numpy()
    dy = synth.grad_output(cfg, T=cfg.T)[:n_tok].float().numpy()
    W_r = synth.router_weight(cfg).float().numpy().T
    shared = None
    if cfg.E_s:
        s_gu, s_down = synth.shared_weights(cfg)
        fs = cfg.E_s * cfg.f
        shared = (s_gu[:fs].float().numpy().T, s_gu[fs:].float().numpy().T,
                  s_down.float().numpy().T)
    bias = synth.zipf_bias(cfg)
    return x, dy, W_r, Wg, Wu, Wd, shared, None if bias is None else bias.numpy()


def _oracle_step(cfg, inp):
    from oracle import moe_ref as ref
    x, dy, W_r, Wg, Wu, Wd, shared, bias = inp
    return ref.layer_forward_backward(x, W_r, Wg, Wu, Wd, dy, cfg.k, cfg.cf, 1, shared=shared,
                                      bias=bias)


def cpu_baseline(cfg, n_tok, w_gu=None, w_down=None, layer=None):
    if w_gu is not None and w_gu.shape[0] != cfg.E:
        w_gu = w_down = None
    inp = _oracle_inputs(cfg, n_tok, w_gu, w_down)
    t = time.perf_counter()
    _oracle_step(cfg, inp)
    dt = time.perf_counter() - t
    return {"value": n_tok / dt, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
            "kind": "oracle",
            "sample": f"one fwd+bwd of the fp64 NumPy oracle on the first {n_tok} tokens of the "
                      f"{cfg.name} workload (all {cfg.E} experts, full d/f), {dt:.1f} s"}


def run_reference(args):
    world, rank, local = dist_env()
    if world > 1 and rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    n_tok = args.cpu_sample_tokens
    if not n_tok:
        if cfg.name == "tiny":
            n_tok = cfg.T
        else:
            # size each step so the whole K+W run stays within ~2 minutes of host time:
            # one calibration step on 32 tokens, then tokens per step in [16, 256]
            probe = _oracle_inputs(cfg, 32)
            t0 = time.perf_counter()
            _oracle_step(cfg, probe)
            per_tok = (time.perf_counter() - t0) / 32
            budget = 120.0 / max(args.steps + args.warmup, 1)
            n_tok = int(min(256, max(16, budget / per_tok)))
    inp = _oracle_inputs(cfg, n_tok)
    for _ in range(args.warmup):
        _oracle_step(cfg, inp)
    t = time.perf_counter()
    for _ in range(args.steps):
        _oracle_step(cfg, inp)
    dt = (time.perf_counter() - t) / max(args.steps, 1)
    v = n_tok / dt
    out = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded N(0,1) tokens, random-init expert/router weights)",
        "impl": "reference",
        "config": {"workload": f"{cfg.name} MoE layer fwd+bwd", "T": cfg.T, "d": cfg.d,
                   "E": cfg.E, "k": cfg.k, "f": cfg.f, "E_shared": cfg.E_s,
                   "capacity_factor": cfg.cf, "parallelism": f"ep{args.gpus}"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                         "kind": "oracle",
                         "sample": f"each step = one fwd+bwd of the fp64 NumPy oracle on the first "
                                   f"{n_tok} tokens of the workload (all experts, full d/f)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ---------------------------------------------------------------------------- NEXT-3 pipeline
def run_pipeline(args):
    """PP x EP executor (paper_2605_05049_b200.pipeline): a stack of --layers MoE layers of the
    config's shape, --micro micro-batches of T/--micro tokens each per step, 1F1B.  value =
    tokens of the step / (max-over-ranks device time of one step); not the headline metric."""
    world, rank, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    from paper_2605_05049_b200 import LayerDims
    from paper_2605_05049_b200.pipeline import PipelineStack
    cfg = synth.CONFIGS[args.config]
    pp, M, Lyr = args.pp, args.micro, args.layers
    ep = world // pp
    stage, e = divmod(rank, ep)
    T_mb = cfg.T // M
    T_r = T_mb // ep
    dims = LayerDims(T_r, cfg.d, cfg.E, cfg.k, cfg.f, cfg.E_s, cfg.cf, ep, e)
    stack = PipelineStack(dims, Lyr, pp, M, device=local, dedup=args.dedup)
    E_l = cfg.E // ep
    dev = torch.device(f"cuda:{local}")
    w_gu, w_down = synth.expert_weights(cfg, range(e * E_l, (e + 1) * E_l), device=dev)
    w_gu_s, w_down_s = synth.shared_weights(cfg, device=dev)
    for l in range(Lyr // pp):
        stack.set_weights(l, synth.router_weight(cfg, device=dev), w_gu, w_down,
                          synth.zipf_bias(cfg), w_gu_s, w_down_s)
    x = synth.tokens(cfg, device=dev).view(M, T_mb, cfg.d)
    dy = synth.grad_output(cfg, device=dev).view(M, T_mb, cfg.d)
    xs = [x[m, e * T_r:(e + 1) * T_r].contiguous() for m in range(M)]
    dys = [dy[m, e * T_r:(e + 1) * T_r].contiguous() for m in range(M)]
    first, last = stage == 0, stage == pp - 1

    def step():
        stack.step(xs if first else None, dys if last else None)
    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(local)
    clocks.start()                 # before the barrier: the ranks enter the loop together
    torch.cuda.synchronize()
    dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    eager = t0.elapsed_time(t1) / args.steps
    graph_ms, graph_note = 0.0, None
    if args.graph:
        # the whole 1F1B step (layer calls + NCCL hand-offs) replayed from one CUDA graph
        try:
            graph = stack.capture(xs if first else None, dys if last else None)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
            dist.barrier()
            t0.record()
            for _ in range(args.steps):
                graph.replay()
            t1.record()
            torch.cuda.synchronize()
            dist.barrier()
            graph_ms = t0.elapsed_time(t1) / args.steps
            # release the captured NCCL work before the contexts and the process group go
            # (keeping the graph alive through close/destroy hung the processes at exit)
            del graph
            torch.cuda.synchronize()
        except Exception as exc:   # reported, the eager number stands
            graph_note = f"capture failed: {type(exc).__name__}: {str(exc)[:200]}"
    tt = torch.tensor([eager, graph_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    eager, graph_ms = tt.tolist()
    ms = graph_ms if (args.graph and graph_ms > 0 and graph_ms < eager) else eager
    # serial per-stage GEMM bound of the step: every stage does M micro-batches of L/PP layers
    rows = M * T_r * cfg.k
    gemm_flops = (Lyr // pp) * 18 * rows * cfg.d * cfg.f
    peaks = measured_peaks()
    if rank == 0:
        print(json.dumps({
            "metric": "PP x EP MoE stack fwd+bwd tokens/s", "value": cfg.T / (ms * 1e-3),
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded N(0,1) tokens, random-init weights)",
            "config": {"workload": f"{cfg.name} {Lyr}-layer MoE stack, 1F1B",
                       "parallelism": f"pp{pp}xep{ep}", "micro_batches": M,
                       "tokens_per_micro_batch": T_mb, "layers": Lyr,
                       "dedup_a2a": args.dedup, "eager_ms_per_step": eager,
                       "graph_ms_per_step": graph_ms or None, "graph_note": graph_note},
            "gpu_launches": None, "clocks": clk,
            "stage_gemm_bound_ms": gemm_flops / (peaks["bf16_sustained"] * 1e12) * 1e3,
            "pipeline_bubble_bound": (pp - 1) / (M + pp - 1),
        }), flush=True)
    stack.close()
    dist.barrier()
    dist.destroy_process_group()


# ---------------------------------------------------------------------------- a2a sweep
def run_a2a(args):
    """Config 5: equal-split all-to-all of a bf16 send buffer, 64 KB .. 1 GB per rank:
    our NVSwitch peer-store dispatch (moe_dispatch, one expert per rank, no capacity; it
    exchanges the counts itself), our static equal-split all-to-all (moe_all_to_all: the same
    layout as NCCL's, no counts round) vs torch.distributed.all_to_all_single (NCCL) with static
    splits, and vs NCCL used with data-dependent splits (counts all-to-all, host read-back,
    variable all-to-all).  Eager and CUDA-graph timings.  Reports busbw (nccl-tests)."""
    world, rank, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    from paper_2605_05049_b200 import _lib as L
    assert world > 1, "--a2a needs torchrun with >= 2 ranks"
    d = 4096
    results = []
    for p in range(16, 31, 1):
        size = 1 << p
        rows = size // (d * 2)
        if rows < world or rows % world:
            d_eff = 512
            rows = size // (d_eff * 2)
        else:
            d_eff = d
        T = rows  # tokens per rank, k=1, E = world (one expert per rank), balanced
        shape = L.make_shape(T, d_eff, world, 1, 128, 0, 0.0, world, rank)
        R = L.moe_recv_rows_max(shape)
        ctx = L.Context(shape, local, 2 * R * d_eff * 2 + T * d_eff * 2 + 8 * 4096)
        from paper_2605_05049_b200.layer import _all_gather_bytes
        ctx.open_peers(_all_gather_bytes(ctx.export_handle()))
        xr = ctx.symm_empty((R, d_eff), torch.bfloat16)
        ra = ctx.symm_empty((world, T // world * d_eff), torch.bfloat16)   # static a2a target
        xs = torch.randn((T, d_eff), device="cuda").to(torch.bfloat16)
        counts = torch.full((world,), T // world, dtype=torch.int32, device="cuda")
        layout = torch.zeros((L.moe_layout_ints(shape),), dtype=torch.int32, device="cuda")
        ref_out = torch.empty_like(xs)
        xsv = xs.view(world, -1)
        for _ in range(3):
            L.moe_dispatch(ctx, xs, counts, layout, xr)
            L.moe_all_to_all(ctx, xsv, ra)
            dist.all_to_all_single(ref_out, xs)
        torch.cuda.synchronize()
        ok = torch.equal(xr[:T], ref_out)
        ok_static = torch.equal(ra.view(-1), ref_out.view(-1))
        # enough calls that the ranks' launch skew after the barrier is amortised
        it = 200 if size <= (16 << 20) else 20
        for _ in range(it):   # clocks up, caches warm
            L.moe_dispatch(ctx, xs, counts, layout, xr)
            L.moe_all_to_all(ctx, xsv, ra)
            dist.all_to_all_single(ref_out, xs)
        dist.barrier(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(it):
            L.moe_dispatch(ctx, xs, counts, layout, xr)
        e.record(); torch.cuda.synchronize()
        t_ours = s.elapsed_time(e) / it
        dist.barrier(); torch.cuda.synchronize()
        s.record()
        for _ in range(it):
            L.moe_all_to_all(ctx, xsv, ra)
        e.record(); torch.cuda.synchronize()
        t_static = s.elapsed_time(e) / it
        dist.barrier(); torch.cuda.synchronize()
        s.record()
        for _ in range(it):
            dist.all_to_all_single(ref_out, xs)
        e.record(); torch.cuda.synchronize()
        t_nccl = s.elapsed_time(e) / it
        # the same `it` calls replayed from CUDA graphs: device time without the host
        # launch path (small messages are launch-bound when issued eagerly)
        def graph_of(fn):
            s2 = torch.cuda.Stream()
            s2.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s2):
                fn()
            torch.cuda.current_stream().wait_stream(s2)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s2):
                for _ in range(it):
                    fn()
            return g
        tg = []
        for fn in (lambda: L.moe_dispatch(ctx, xs, counts, layout, xr),
                   lambda: dist.all_to_all_single(ref_out, xs),
                   lambda: L.moe_all_to_all(ctx, xsv, ra)):
            try:
                g = graph_of(fn)
                g.replay()
                dist.barrier(); torch.cuda.synchronize()
                s.record()
                g.replay()
                e.record(); torch.cuda.synchronize()
                tg.append(s.elapsed_time(e) / it)
                del g
            except Exception:   # capture unsupported: report eager only
                tg.append(float("nan"))
        ok = ok and torch.equal(xr[:T], ref_out)
        # NCCL as an MoE dispatch with data-dependent sizes uses it: all-to-all of the counts,
        # the splits read back on the host, then the variable-size all-to-all
        send_counts = counts.clone()
        recv_counts = torch.empty_like(send_counts)

        def nccl_dynamic():
            dist.all_to_all_single(recv_counts, send_counts)
            out_splits = recv_counts.tolist()
            dist.all_to_all_single(ref_out, xs, output_split_sizes=out_splits,
                                   input_split_sizes=[T // world] * world)
        nccl_dynamic()
        dist.barrier(); torch.cuda.synchronize()
        s.record()
        for _ in range(it):
            nccl_dynamic()
        e.record(); torch.cuda.synchronize()
        t_dyn = s.elapsed_time(e) / it
        ok = ok and torch.equal(xr[:T], ref_out)
        ok_static = ok_static and torch.equal(ra.view(-1), ref_out.view(-1))
        v = torch.tensor([t_ours, t_nccl, *tg, t_dyn, t_static], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        t_ours, t_nccl, tg_ours, tg_nccl, tg_static, t_dyn, t_static = v.tolist()
        nbytes = T * d_eff * 2
        bus = (world - 1) / world
        results.append({"bytes_per_rank": nbytes, "bitwise_equal_nccl": bool(ok),
                        "static_bitwise_equal_nccl": bool(ok_static),
                        "static_ms": t_static, "static_graph_ms": tg_static,
                        "static_busbw_GBs": nbytes / (t_static * 1e-3) / 1e9 * bus,
                        "static_graph_busbw_GBs": nbytes / (tg_static * 1e-3) / 1e9 * bus,
                        "ours_ms": t_ours, "nccl_ms": t_nccl,
                        "ours_graph_ms": tg_ours, "nccl_graph_ms": tg_nccl,
                        "nccl_dynamic_ms": t_dyn,
                        "ours_busbw_GBs": nbytes / (t_ours * 1e-3) / 1e9 * bus,
                        "nccl_busbw_GBs": nbytes / (t_nccl * 1e-3) / 1e9 * bus,
                        "ours_graph_busbw_GBs": nbytes / (tg_ours * 1e-3) / 1e9 * bus,
                        "nccl_graph_busbw_GBs": nbytes / (tg_nccl * 1e-3) / 1e9 * bus})
        ctx.close()
    if rank == 0:
        print(json.dumps({"metric": "dispatch all-to-all busbw vs NCCL", "n_gpus": world,
                          "unit": "GB/s", "nvlink_peak_GBs": 900, "sweep": results}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_gemm_compare(args):
    """Expert FFN fwd+bwd GEMMs of one rank (balanced rows, EP = 1) through libmoe vs the same
    contractions issued to cuBLAS via torch (per-expert matmuls + elementwise SwiGLU), in the
    same process and power state; plus one large square cuBLAS GEMM as the box's dense-bf16
    reference.  Context for the roofline fraction, not a bench line."""
    torch.cuda.set_device(0)
    from paper_2605_05049_b200 import _lib as L
    cfg = synth.CONFIGS[args.config]
    E, d, f = cfg.E, cfg.d, cfg.f
    rows = cfg.T * cfg.k // E
    if args.gemm_experts:   # one EP rank's share: E_l experts of `rows` rows
        E = args.gemm_experts
        rows = args.gemm_rows or rows
        cfg = synth.MoEConfig(f"{cfg.name}_E{E}_r{rows}", T=rows * E, d=d, E=E, k=1, f=f, cf=0.0)
    R = rows * E
    dev = torch.device("cuda:0")
    shape = L.make_shape(cfg.T, d, E, cfg.k, f, 0, 0.0, 1, 0)
    ctx = L.Context(shape, 0, 4096)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    bf = torch.bfloat16
    xr = torch.randn((R, d), device=dev, generator=g).to(bf)
    dout = torch.randn((R, d), device=dev, generator=g).to(bf)
    w_gu, w_down = synth.expert_weights(cfg, range(E), device=dev)
    group_rows = torch.full((E,), rows, dtype=torch.int32, device=dev)
    g_u_h = torch.empty((R, 3 * f), dtype=bf, device=dev)
    out = torch.empty((R, d), dtype=bf, device=dev)
    dgu = torch.empty((R, 2 * f), dtype=bf, device=dev)
    dxr = torch.empty((R, d), dtype=bf, device=dev)
    dw_gu = torch.empty((E, 2 * f, d), dtype=torch.float32, device=dev)
    dw_down = torch.empty((E, d, f), dtype=torch.float32, device=dev)

    def ours():
        L.moe_expert_ffn(ctx, xr, group_rows, E, R, f, w_gu, w_down, g_u_h, out)
        L.moe_expert_ffn_bwd(ctx, xr, group_rows, E, R, f, w_gu, w_down, g_u_h, dout, dgu, dxr,
                             dw_gu, dw_down)

    # cuBLAS gets the six contractions only (its SwiGLU / dSwiGLU inputs precomputed): the
    # libmoe side also runs its fused epilogues, so the comparison favours cuBLAS
    H_all = g_u_h[:, 2 * f:].contiguous()
    dGU_all = torch.randn((R, 2 * f), device=dev, generator=g).to(bf)
    o_buf = torch.empty((rows, d), dtype=bf, device=dev)
    gu_buf = torch.empty((rows, 2 * f), dtype=bf, device=dev)
    dh_buf = torch.empty((rows, f), dtype=bf, device=dev)

    def cublas():
        for e in range(E):
            X = xr[e * rows:(e + 1) * rows]
            dO = dout[e * rows:(e + 1) * rows]
            H = H_all[e * rows:(e + 1) * rows]
            dGU = dGU_all[e * rows:(e + 1) * rows]
            torch.mm(X, w_gu[e].t(), out=gu_buf)
            torch.mm(H, w_down[e].t(), out=o_buf)
            torch.mm(dO, w_down[e], out=dh_buf)
            torch.mm(dGU, w_gu[e], out=o_buf)
            torch.mm(dO.t(), H, out_dtype=torch.float32)
            torch.mm(dGU.t(), X, out_dtype=torch.float32)

    def timeit(fn, n):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    flops = 18.0 * R * d * f
    res = {"config": cfg.name, "rows_per_expert": rows, "experts": E, "flops": flops}
    n = 8192
    A = torch.randn((n, n), device=dev, generator=g).to(bf)
    B = torch.randn((n, n), device=dev, generator=g).to(bf)
    clocks = ClockSampler(0)
    t = {}
    for name, fn, it in (("ours", ours, args.steps), ("cublas", cublas, args.steps),
                         ("square", lambda: torch.mm(A, B), 200)):
        clocks.start()
        t[name] = timeit(fn, it)
        res[f"clocks_{name}"] = clocks.stop()
    t_ours, t_cub, t_sq = t["ours"], t["cublas"], t["square"]
    res.update(ours_ms=t_ours, cublas_ms=t_cub, ours_tflops=flops / t_ours / 1e9,
               cublas_tflops=flops / t_cub / 1e9, cublas_square8192_tflops=2 * n ** 3 / t_sq / 1e9)
    print(json.dumps(res), flush=True)
    ctx.close()


def run_migrate_bench(args):
    """NEXT-2 migration cost (Table): the worst case of the
    paper's table -- every expert moves (placement rotated by one rank) -- with each expert's
    whole training state: bf16 weights (2 B/param), fp32 weight gradients (4), an fp32 master
    copy and two fp32 Adam moments (12): 18 B per parameter (>= the paper's 16).  One
    moe_migrate launch per state tensor, CUDA events on the stream, max over ranks."""
    world, rank, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    from paper_2605_05049_b200 import LayerDims, MoELayer
    from paper_2605_05049_b200 import _lib as L
    assert world > 1, "--migrate-bench needs torchrun with >= 2 ranks"
    cfg = synth.CONFIGS[args.config]
    E_l, n_par = cfg.E // world, 3 * cfg.d * cfg.f
    dims = LayerDims(cfg.T // world, cfg.d, cfg.E, cfg.k, cfg.f, cfg.E_s, cfg.cf, world, rank)
    layer = MoELayer(dims, device=local, migratable=True, expert_state_bytes=12 * n_par)
    opt = [layer.expert_state(nm, (n_par,), torch.float32) for nm in ("master", "m", "v")]
    dev = torch.device(f"cuda:{local}")
    w_gu, w_down = synth.expert_weights(cfg, range(rank * E_l, (rank + 1) * E_l), device=dev)
    layer.set_weights(synth.router_weight(cfg, device=dev), w_gu, w_down)
    for t in opt:
        t.normal_()
    layer.dw_gu.normal_()
    layer.dw_down.normal_()
    rot = [(s + E_l) % cfg.E for s in range(cfg.E)]       # every expert to the next rank
    times = []
    for it in range(args.warmup + args.steps):
        new = [rot[s] for s in layer.placement]
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        old = list(layer.placement)
        nxt = 1 - layer._cur
        for bufs in layer._states.values():
            L.moe_migrate(layer.ctx, old, new, bufs[layer._cur], bufs[nxt])
        b.record()
        torch.cuda.synchronize()
        layer._cur = nxt
        layer.placement = new
        layer.ctx.set_placement(new)
        if it >= args.warmup:
            times.append(a.elapsed_time(b))
    ms = torch.tensor([float(np.median(times))], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    state_bytes = E_l * n_par * (2 + 4 + 12)            # per rank, all moved
    paper_bytes = 48 * E_l * cfg.d * cfg.f               # PAPER.md:648 per rank (16 B/param)
    if rank == 0:
        print(json.dumps({
            "metric": "expert migration time (every expert moves, full training state)",
            "n_gpus": world, "config": cfg.name, "experts_per_rank": E_l,
            "bytes_per_param": 18, "bytes_per_rank": state_bytes, "ms": ms,
            "gb_per_s_per_rank": state_bytes / (ms * 1e-3) / 1e9,
            "paper_table_bytes_per_rank": paper_bytes,
            "paper_model_ms_at_50GBps": paper_bytes / 50e9 * 1e3,
            "ours_ms_scaled_to_16B_per_param": ms * 16 / 18,
            "note": "one moe_migrate launch per state tensor (weights x2, grads x2, master, m, "
                    "v): barrier, peer stores into the new owners' other buffer half, flags"}),
              flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.migrate_bench:
        run_migrate_bench(args)
    elif args.gemm_compare:
        run_gemm_compare(args)
    elif args.pp > 1:
        run_pipeline(args)
    elif args.a2a:
        run_a2a(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

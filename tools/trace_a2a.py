"""Phase latencies of one small moe_dispatch (globaltimer stamps, -DMOE_TRACE build).

    python tools/trace_a2a.py --build          # here: builds paper_2605_05049_b200/libmoe_trace.so
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/trace_a2a.py   # on the GPU box
Prints per rank: launch gap, counts round, tables, copy, signal, data round (microseconds).
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_05049_b200")
TRACE_LIB = os.path.join(PKG, "libmoe_trace.so")


def build():
    sys.path.insert(0, PKG)
    import build as b
    objdir = os.path.join(PKG, "build", "trace")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in b.SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        subprocess.run([b.NVCC, *b.FLAGS, "-DMOE_TRACE", "-c", os.path.join(b.CSRC, src), "-o", obj],
                       check=True)
        objs.append(obj)
    subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                    TRACE_LIB, *objs, "-Xcompiler", "-fPIC"], check=True)
    print(TRACE_LIB)


def run(args):
    os.environ["MOE_LIB"] = TRACE_LIB
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    world, rank = dist.get_world_size(), dist.get_rank()
    from paper_2605_05049_b200 import _lib as L
    from paper_2605_05049_b200.layer import _all_gather_bytes
    d = args.width
    T = max(args.bytes // (d * 2), world)
    shape = L.make_shape(T, d, world, 1, 128, 0, 0.0, world, rank)
    R = L.moe_recv_rows_max(shape)
    ctx = L.Context(shape, local, 2 * R * d * 2 + 4 * 4096)
    ctx.open_peers(_all_gather_bytes(ctx.export_handle()))
    xr = ctx.symm_empty((R, d), torch.bfloat16)
    xs = torch.randn((T, d), device="cuda").to(torch.bfloat16)
    counts = torch.full((world,), T // world, dtype=torch.int32, device="cuda")
    layout = torch.zeros((L.moe_layout_ints(shape),), dtype=torch.int32, device="cuda")
    for _ in range(args.iters):
        L.moe_dispatch(ctx, xs, counts, layout, xr)
    torch.cuda.synchronize()
    tr = (ctypes.c_ulonglong * (64 * 8))()
    fn = L._lib.moe_debug_trace
    fn.argtypes = [ctypes.c_void_p]
    assert fn(ctypes.cast(tr, ctypes.c_void_p)) == 0
    t = [list(tr[8 * i:8 * i + 8]) for i in range(64)]
    # epochs 1..iters map to rows epoch % 64; take the last min(iters, 63) - 1 calls
    last = args.iters
    rows = [(e, t[e % 64]) for e in range(max(2, last - 60), last + 1)]
    import statistics as st
    names = {"gap_prev_end_to_start": lambda e, r: r[0] - t[(e - 1) % 64][5],
             "counts_published": lambda e, r: r[6] - r[0],
             "counts_round": lambda e, r: r[1] - r[0], "tables": lambda e, r: r[2] - r[1],
             "copy": lambda e, r: r[3] - r[2], "to_last_block": lambda e, r: r[4] - r[3],
             "data_round_wait": lambda e, r: r[5] - r[4], "total": lambda e, r: r[5] - r[0]}
    out = {"rank": rank, "bytes": T * d * 2, "d": d, "calls": len(rows)}
    for n, f in names.items():
        out[n] = st.median(f(e, r) for e, r in rows) / 1e3
    outs = [None] * world
    dist.all_gather_object(outs, out)
    if rank == 0:
        for o in outs:
            print(json.dumps(o))
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--bytes", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--width", type=int, default=512)
    a = ap.parse_args()
    build() if a.build else run(a)

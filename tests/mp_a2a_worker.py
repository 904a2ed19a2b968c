"""torchrun worker: the NVSwitch all-to-alls alone, with ORIGIN-ENCODED payloads (SURVEY.md
§4.1): every send row carries (source rank, send row) as exact small integers
in its bf16 elements, so a misrouted, duplicated, dropped or torn row is detected exactly.

Per rank, against the oracle's receive layout (oracle.moe_ref.recv_layout) of the gathered
[EP x E] count matrix:
  * moe_dispatch: every received row equals the expected source row bit for bit; padding
    rows of every 128-aligned segment are zero; the layout record equals the oracle's;
  * moe_dispatch_bwd(moe_dispatch(xs)) == xs on the sent rows (involution);
  * moe_dispatch_range over two slot ranges == moe_dispatch, bit for bit;
  * the same after a random expert placement (moe_ctx_set_placement).
Counts are seeded, ragged, include zeros and one source that sends nothing to anyone.
Prints one JSON line on rank 0: {"ok": bool, "checks": {...}}.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from tests import mp_common  # noqa: E402


def encoded_rows(rank, n, d):
    """Row i of source `rank`: [rank, i // 128, i % 128, (7 rank + 3 i + c) % 251 - 125 ...];
    every value is an integer of magnitude < 256, exact in bf16."""
    i = torch.arange(n, dtype=torch.int64)[:, None]
    c = torch.arange(d, dtype=torch.int64)[None, :]
    v = (7 * rank + 3 * i + c) % 251 - 125
    v[:, 0] = rank
    v[:, 1] = (i // 128)[:, 0]
    v[:, 2] = (i % 128)[:, 0]
    return v.to(torch.float32).to(torch.bfloat16)


def main():
    local, shared = mp_common.init()
    ep, rank = dist.get_world_size(), dist.get_rank()
    from paper_2605_05049_b200 import _lib as L
    from paper_2605_05049_b200.layer import _all_gather_bytes
    from oracle import moe_ref as ref

    T_r, d, k = 300, 256, 2
    E = 4 * ep
    E_l = E // ep
    shape = L.make_shape(T_r, d, E, k, 128, 0, 0.0, ep, rank)
    R = L.moe_recv_rows_max(shape)
    ctx = L.Context(shape, local, 2 * R * d * 2 + 2 * T_r * k * d * 2 + ep * 3 * 128 * 16 + 8 * 4096)
    ctx.open_peers(_all_gather_bytes(ctx.export_handle()))
    xr = ctx.symm_empty((R, d), torch.bfloat16)
    xr2 = ctx.symm_empty((R, d), torch.bfloat16)
    dxs = ctx.symm_empty((T_r * k, d), torch.bfloat16)
    lay_n = L.moe_layout_ints(shape)

    # seeded ragged counts: row r of the [EP, E] matrix, sum <= T_r * k; source 1 sends nothing
    rng = np.random.default_rng(2024)
    cm = np.zeros((ep, E), np.int64)
    for r in range(ep):
        if r == 1:
            continue
        w = rng.random(E) * (rng.random(E) < 0.75)
        cm[r] = np.floor(w / max(w.sum(), 1e-9) * rng.integers(T_r, T_r * k + 1)).astype(np.int64)
    counts = torch.tensor(cm[rank], dtype=torch.int32, device="cuda")
    n_send = int(cm[rank].sum())
    xs = torch.zeros((T_r * k, d), dtype=torch.bfloat16, device="cuda")
    xs[:n_send] = encoded_rows(rank, n_send, d).cuda()
    checks = {}

    def sync():
        torch.cuda.synchronize()
        dist.barrier()

    def check_layout(tag, xr_t, layout, placement):
        lay = layout.cpu().numpy()
        want = ref.recv_layout(cm, ep, align=128, placement=placement)[rank]
        ok = bool((lay[:ep * E].reshape(ep, E) == cm).all())
        ok &= bool((lay[ep * E:ep * E + E_l] == want["expert_rows"]).all())
        ok &= bool((lay[ep * E + E_l:] == want["seg_base"]).all())
        checks[f"{tag}_layout"] = ok
        got = xr_t.cpu()
        rows_ok = True
        for el in range(E_l):
            e = int(want["expert"][el])
            for r in range(ep):
                n = int(cm[r, e])
                if n == 0:
                    continue
                off = int(cm[r, :e].sum())       # send-layout offset of expert e on source r
                exp = encoded_rows(r, off + n, d)[off:]
                b = int(want["src_base"][el][r])
                rows_ok &= bool(torch.equal(got[b:b + n], exp))
            lo = int(want["seg_base"][el]) + int(want["expert_rows"][el])
            hi = int(want["seg_base"][el + 1])
            rows_ok &= bool((got[lo:hi] == 0).all())
        checks[f"{tag}_rows"] = rows_ok

    for tag, placement in (("contiguous", None), ("placed", np.random.default_rng(7).permutation(E))):
        if placement is not None:
            ctx.set_placement([int(v) for v in placement])
        layout = torch.zeros((lay_n,), dtype=torch.int32, device="cuda")
        xr.fill_(7.0)   # stale contents must be overwritten or zeroed
        sync()          # a peer's stores into my buffer must not race my own fill
        L.moe_dispatch(ctx, xs, counts, layout, xr)
        torch.cuda.synchronize()
        check_layout(tag, xr, layout, placement)
        dxs.zero_()
        sync()
        L.moe_dispatch_bwd(ctx, xr, layout, dxs)
        torch.cuda.synchronize()
        checks[f"{tag}_involution"] = bool(torch.equal(dxs[:n_send], xs[:n_send]))
        layout2 = torch.zeros_like(layout)
        xr2.fill_(7.0)
        sync()
        half = max(1, E_l // 2)
        L.moe_dispatch_range(ctx, xs, counts, layout2, xr2, 0, half)
        L.moe_dispatch_range(ctx, xs, None, layout2, xr2, half, E_l)
        torch.cuda.synchronize()
        used = int(layout2[ep * E + E_l + E_l].item())
        checks[f"{tag}_ranges"] = bool(torch.equal(layout2, layout) and
                                       torch.equal(xr2[:used], xr[:used]))
    # moe_all_to_all (static equal splits, config 5): the transpose law against the oracle's
    # brute-force flat_all_to_all on origin-encoded chunks, twice (epoch reuse)
    n_chunk = 3 * 128
    send = encoded_rows(rank, ep * n_chunk, 8).reshape(ep, n_chunk * 8).cuda()
    ra = ctx.symm_empty((ep, n_chunk * 8), torch.bfloat16)
    allsend = [encoded_rows(r, ep * n_chunk, 8).reshape(-1).float().numpy() for r in range(ep)]
    want = ref.flat_all_to_all(allsend)[rank]
    ok = True
    for _ in range(2):
        sync()
        L.moe_all_to_all(ctx, send, ra)
        torch.cuda.synchronize()
        ok &= bool(np.array_equal(ra.float().cpu().numpy().reshape(-1), want))
    checks["static_all_to_all"] = ok
    st = ctx.device_error()
    flags = torch.tensor([int(all(checks.values())), st], device="cuda")
    allf = mp_common.gather(flags)
    if rank == 0:
        res = {"ep": ep, "ok": all(int(f[0]) == 1 and int(f[1]) == 0 for f in allf),
               "per_rank": [[int(f[0]), int(f[1])] for f in allf], "checks_rank0": checks}
        print(json.dumps(res), flush=True)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

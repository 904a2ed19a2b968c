"""World-size-2 gloo tests (CPU) of the host-side multi-process logic: the symmetric-heap
handle exchange MoELayer uses, the token/expert sharding, and the max-over-ranks timing
reduction of bench.py -- everything of the N>1 path that does not need a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_05049_b200.layer import _all_gather_bytes
        import synth
        payload = bytes([rank * 16 + i for i in range(64)])      # a 64-byte "IPC handle"
        allh = _all_gather_bytes(payload)
        ok_handles = allh == b"".join(bytes([r * 16 + i for i in range(64)]) for r in range(world))
        # token / expert sharding used by bench.py and the multi-GPU worker
        cfg = synth.CONFIGS["tiny"]
        T_r, E_l = cfg.T // world, cfg.E // world
        x = synth.tokens(cfg)
        mine = x[rank * T_r:(rank + 1) * T_r]
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine.contiguous())
        ok_shard = torch.equal(torch.cat(parts), x)
        experts = list(range(rank * E_l, (rank + 1) * E_l))
        allex = [None] * world
        dist.all_gather_object(allex, experts)
        ok_experts = sorted(sum(allex, [])) == list(range(cfg.E))
        # max over ranks of per-rank step times (bench.py timing rule)
        t = torch.tensor([1.0 + rank, 5.0 - rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok_max = t.tolist() == [float(world), 5.0]
        q.put((rank, ok_handles, ok_shard, ok_experts, ok_max))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert all(r[1:]), r


def test_oracle_ep_ranks_partition_the_layer():
    """The oracle's EP simulation: per-rank plans partition every kept slot exactly once
    and the receive layouts of all owners cover exactly the kept rows (EP=2, 4, 8)."""
    import synth
    from oracle import moe_ref as ref
    T, E, k = 512, 8, 2
    idx, _ = ref.route(synth.random_logits(T, E, seed=99).numpy(), k)
    for ep in (2, 4, 8):
        plan = ref.dispatch_plan(idx, E, ep, ref.capacity(1.0, k, T // ep, E), align=128)
        kept = plan["recv_row"] >= 0
        for q in range(ep):
            rows = plan["recv_row"][kept & (plan["owner"] == q)]
            lay = plan["layouts"][q]
            assert len(set(rows.tolist())) == rows.size == lay["expert_rows"].sum()
            # every row falls inside its expert's segment, before the padding
            for el in range(E // ep):
                seg0, seg1 = lay["seg_base"][el], lay["seg_base"][el] + lay["expert_rows"][el]
                m = kept & (idx == q * (E // ep) + el)
                assert ((plan["recv_row"][m] >= seg0) & (plan["recv_row"][m] < seg1)).all()


def _dedup_worker(rank, world, port, q):
    """One EP rank of the deduplicated exchange (reading R18) with gloo standing in for the
    NVSwitch stores: local pairs from the rank's own shard, the pair-count exchange, token rows
    sent once per (token, owner) pair, and the owner's expand into the plain receive layout."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import dedup as dd
        from oracle import moe_ref as ref
        T, E, k, d = 256, 16, 4, 8
        T_r, E_l = T // world, E // world
        idx, gates = ref.route(synth.random_logits(T, E, seed=5).numpy(), k)
        C = ref.capacity(1.0, k, T_r, E)
        mine = slice(rank * T_r, (rank + 1) * T_r)
        pos = ref.positions(idx[mine], E, C)                            # this rank only
        pr = dd.pairs(pos["dest_row"], idx[mine], np.arange(E), E_l, world)
        ntok = torch.tensor(pr["ntok"], dtype=torch.int64)
        allnt = [torch.empty_like(ntok) for _ in range(world)]
        dist.all_gather(allnt, ntok)                                   # the pair-count exchange
        ntok_all = torch.stack(allnt).numpy()
        full = dd.plan(idx, gates, E, world, C, align=128)            # single-process reference
        ok_counts = (ntok_all == full["ntok_all"]).all()
        x = np.random.default_rng(1).standard_normal((T, d))
        send = [x[mine][pr["tslot"][:, qq] >= 0] for qq in range(world)]   # tslot order
        recv = [None] * world
        dist.all_gather_object(recv, send)                            # gloo as the transport
        xt = np.concatenate([recv[r][rank] for r in range(world)])   # (source, tslot) order
        n_rows = int(full["base"]["layouts"][rank]["seg_base"][-1])
        xr = dd.expand(xt, full["rlist"][rank], n_rows)
        plain = np.zeros((n_rows, d))
        b = full["base"]
        t, j = np.nonzero((b["owner"] == rank) & (b["recv_row"] >= 0))
        plain[b["recv_row"][t, j]] = x[t]
        ok_xr = np.array_equal(xr, plain)
        q.put((rank, bool(ok_counts), bool(ok_xr)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_dedup_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dedup_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert all(r[1:]), r

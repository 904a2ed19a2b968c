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
        # tests/mp_common.gather (the shared-GPU workers' result gather over gloo)
        from tests import mp_common
        g = mp_common.gather(torch.full((3,), float(rank)))
        ok_gather = [t.tolist() for t in g] == [[float(r)] * 3 for r in range(world)]
        # the symmetric-allocation fingerprint exchange: identical sequences agree
        fp = (1469598103934665603 ^ 12345).to_bytes(8, "little")
        ok_fp = _all_gather_bytes(fp) == fp * world
        q.put((rank, ok_handles, ok_shard, ok_experts, ok_max, ok_gather, ok_fp))
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


class _ToyLayer:
    """CPU stand-in for MoELayer with the interface PipelineStack uses (bf16 activations):
    y = bf16(a*x + 1), dx = bf16(a*dy), and a 'weight gradient' dw = sum(dy*x) in fp32,
    overwritten by the first backward and accumulated by the others."""

    def __init__(self, dims, device=None, group=None, fused=True, dedup=False, migratable=None):
        self.dims = dims
        self.fs = 0
        self.a = 1.0
        self.y = torch.empty(dims.T_local, dims.d, dtype=torch.bfloat16)
        self.dx = torch.empty(dims.T_local, dims.d, dtype=torch.bfloat16)
        self.dw_r = torch.zeros(1)
        self.dw_gu = torch.zeros(1)
        self.dw_down = torch.zeros(1)
        self.w_r = self.w_gu = self.w_down = self.bias = self.w_gu_s = self.w_down_s = None

    def set_weights(self, w_r, w_gu, w_down, bias=None, w_gu_s=None, w_down_s=None):
        self.a = float(w_r)

    def forward(self, x):
        self.x = x
        self.y.copy_(self.a * x.float() + 1.0)
        return self.y

    def backward(self, dy, accumulate=False):
        v = (dy.float() * self.x.float()).sum().reshape(1)
        self.dw_r.copy_(self.dw_r + v if accumulate else v)
        self.dx.copy_(self.a * dy.float())
        return self.dx

    def close(self):
        pass


def _pipe_worker(rank, world, port, q, pp=2, M=5):
    """PP=2 x EP=2 over gloo: the 1F1B op lists from libmoe, stage-to-stage activations and
    gradients, per-micro-batch activation contexts and gradient accumulation -- bitwise
    against the same bf16 arithmetic done sequentially."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_05049_b200 import LayerDims
        from paper_2605_05049_b200.pipeline import PipelineStack
        ep = world // pp
        L, T, d = 4, 3, 4
        stage, e = divmod(rank, ep)
        per = L // pp
        dims = LayerDims(T, d, 4, 1, 8, 0, 1.0, ep, e)
        st = PipelineStack(dims, L, pp, M, device=None, layer_cls=_ToyLayer)
        a = [1.5, -0.5, 2.0, 0.25]                       # per global layer
        for l in range(per):
            st.set_weights(l, a[stage * per + l], None, None)
        g = torch.Generator().manual_seed(7)
        xs = [(torch.randn(T, d, generator=g) + e).bfloat16() for _ in range(M)]
        dys = [(torch.randn(T, d, generator=g) - e).bfloat16() for _ in range(M)]
        ys, dxs = st.step(xs if stage == 0 else None, dys if stage == pp - 1 else None)
        # the same arithmetic, layer by layer, on this EP index's tokens
        hs = [[x] for x in xs]
        gs = [[None] * (L + 1) for _ in range(M)]
        for m in range(M):
            for l in range(L):
                hs[m].append((a[l] * hs[m][l].float() + 1.0).bfloat16())
            gs[m][L] = dys[m]
            for l in reversed(range(L)):
                gs[m][l] = (a[l] * gs[m][l + 1].float()).bfloat16()
        ok = True
        if stage == pp - 1:
            ok &= all(torch.equal(ys[m], hs[m][L]) for m in range(M))
        if stage == 0:
            ok &= all(torch.equal(dxs[m], gs[m][0]) for m in range(M))
        for l in range(per):
            gl = stage * per + l
            want = torch.zeros(1)
            for m in range(M):
                v = (gs[m][gl + 1].float() * hs[m][gl].float()).sum().reshape(1)
                want = v if m == 0 else want + v
            ok &= torch.equal(st.grads(l)[0], want)
        ok &= st.n_slots == min(pp - stage, M)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pp,M", [(2, 5), (4, 2), (4, 6)])
def test_gloo_pipeline(pp, M):
    """PP x EP over gloo with 4 ranks: PP2 x EP2 (M = 5), PP4 x EP1 with fewer micro-batches
    than stages (M = 2: the in-flight bound is M) and with more (M = 6)."""
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_worker, args=(r, world, port, q, pp, M))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        assert r[1], r

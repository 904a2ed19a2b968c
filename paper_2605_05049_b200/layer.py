"""One expert-parallel MoE layer (forward + backward) composed from the C-ABI calls.

This module only allocates buffers (PyTorch device memory and the ctx's symmetric
heap) and issues the libmoe entry points in the order of SURVEY.md §3.3 / §3.4:

  forward : moe_router_logits -> moe_route -> moe_permute -> moe_dispatch ->
            moe_expert_ffn (routed; + shared experts as one group) -> moe_combine
  backward: moe_combine_bwd -> moe_expert_ffn_bwd -> moe_dispatch_bwd ->
            (shared moe_expert_ffn_bwd) -> moe_route_bwd -> moe_router_logits_bwd ->
            moe_permute_bwd

Experts are sharded contiguously (expert e on rank e // (E/EP)) and
tokens are data-parallel (T/EP rows per rank).  With EP > 1 the ranks exchange
their symmetric-heap handles over torch.distributed once at construction.
"""
from __future__ import annotations

import dataclasses

import os

import torch

from . import _lib as L


@dataclasses.dataclass
class LayerDims:
    T_local: int
    d: int
    E: int
    k: int
    f: int
    E_shared: int = 0
    capacity_factor: float = 1.25
    ep_size: int = 1
    ep_rank: int = 0


def _all_gather_bytes(payload: bytes, group=None) -> bytes:
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor(list(payload), dtype=torch.uint8)
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return b"".join(bytes(o.cpu().tolist()) for o in outs)


class MoELayer:
    # extra symmetric-heap room (tests/guard.py puts canary allocations between the buffers)
    extra_heap_bytes = 0

    def __init__(self, dims: LayerDims, device: int = 0, group=None, fused: bool = True,
                 dedup: bool = False, migratable=None, expert_state_bytes: int = 0):
        """fused=True uses the compute+all-to-all entry points (moe_expert_ffn_combine,
        moe_expert_ffn_bwd_dispatch); False issues the step-by-step calls (same results).
        dedup (k > 1; NEXT-4, reading R18): one row per (token, owner) pair on NVLink.
          "dispatch" (or True): the dispatch-direction all-to-alls (dispatch, combine_bwd) are
              deduplicated; combine and dispatch_bwd stay the per-slot transfers fused into the
              GEMM2 / dgrad-2 epilogues (hidden under the GEMMs); results bit-identical to the
              plain path.
          "all": also the reverse direction, as owner-side pair reductions (one extra bf16
              rounding of y and dx).
        migratable (default: EP > 1): the experts' weights and fp32 weight gradients live in
            the symmetric heap, double-buffered, so migrate() can push them to their new owners
            over the peer maps (moe_migrate); expert_state_bytes reserves heap room for more
            per-expert state registered with expert_state() (e.g. optimizer moments)."""
        self.dims = dims
        self.group = group
        self.fused = fused
        mode = "dispatch" if dedup is True else (dedup or None)
        if mode not in (None, "dispatch", "all"):
            raise ValueError(f"dedup must be False, True, 'dispatch' or 'all', got {dedup!r}")
        self.dedup_mode = mode if dims.k > 1 else None
        self.dedup = self.dedup_mode is not None
        self.overlap = True   # shared-expert GEMMs beside dispatch / combine_bwd (E_s > 0)
        self._side = None
        self.placement = list(range(dims.E))   # expert -> global slot (contiguous at start)
        self.loads = None
        self.device = torch.device(f"cuda:{device}")
        self.shape = L.make_shape(dims.T_local, dims.d, dims.E, dims.k, dims.f, dims.E_shared,
                                  dims.capacity_factor, dims.ep_size, dims.ep_rank)
        if L.moe_layout_ints(self.shape) < 0:
            raise ValueError(f"invalid MoE dims {dims}")
        T, d, k, E, f = dims.T_local, dims.d, dims.k, dims.E, dims.f
        self.E_l = E // dims.ep_size
        self.R = L.moe_recv_rows_max(self.shape)
        R = self.R
        heap = 2 * (R * d * 2) + 2 * (max(T * k, 1) * d * 2) + 4 * 4096
        if self.dedup:
            self.tok_max = max(L.moe_dedup_token_rows_max(self.shape), 1)
            self.pair_max = max(L.moe_dedup_pair_rows_max(self.shape), 1)
            heap += self.tok_max * (d * 2 + 8 * k) + self.pair_max * 4 * k + 4 * 4096
        heap += self.extra_heap_bytes
        self.migratable = dims.ep_size > 1 if migratable is None else bool(migratable)
        f32b = 4
        if self.migratable:
            per_expert = 3 * d * f * (2 + f32b)            # bf16 weights + fp32 gradients
            heap += 2 * (self.E_l * per_expert + 4 * 256)
            heap += 2 * (self.E_l * int(expert_state_bytes)) + 64 * 1024
        torch_before = torch.cuda.memory_allocated(self.device)
        self.ctx = L.Context(self.shape, device, heap)
        if dims.ep_size > 1:
            handles = _all_gather_bytes(self.ctx.export_handle(), group)
            self.ctx.open_peers(handles)
        # symmetric (peer-written) buffers -- same allocation order on every rank
        self.xr = self.ctx.symm_empty((R, d), torch.bfloat16)
        self.dout_r = self.ctx.symm_empty((R, d), torch.bfloat16)
        self.ys = self.ctx.symm_empty((max(T * k, 1), d), torch.bfloat16)
        self.dxs = self.ctx.symm_empty((max(T * k, 1), d), torch.bfloat16)
        dev = self.device
        bf, f32, i32 = torch.bfloat16, torch.float32, torch.int32
        if self.dedup:
            # owner side (peer-written): token rows (x in the forward, dy in the backward) and
            # each pair's slot lists; source side: dgpart (the pair partials reuse ys / dxs)
            EP = dims.ep_size
            self.xt = self.ctx.symm_empty((self.tok_max, d), torch.bfloat16)
            self.rlist = self.ctx.symm_empty((self.tok_max, k), torch.int32)
            self.glist = self.ctx.symm_empty((self.tok_max, k), torch.float32)
            self.dgpart = self.ctx.symm_empty((self.pair_max, k), torch.float32)
            self.pdest = torch.empty((T, EP), dtype=i32, device=dev)
            self.ntok = torch.empty((EP,), dtype=i32, device=dev)
            self.dlayout = torch.zeros((EP * EP,), dtype=i32, device=dev)
            self.dg_own = torch.empty((self.tok_max, k), dtype=f32, device=dev)
        self.logits = torch.empty((T, E), dtype=f32, device=dev)
        self.topk_idx = torch.empty((T, k), dtype=i32, device=dev)
        self.gates = torch.empty((T, k), dtype=f32, device=dev)
        self.counts = torch.empty((E,), dtype=i32, device=dev)
        self.dest_row = torch.empty((T, k), dtype=i32, device=dev)
        self.xs = torch.empty((max(T * k, 1), d), dtype=bf, device=dev)
        self.layout = torch.zeros((L.moe_layout_ints(self.shape),), dtype=i32, device=dev)
        eo = L.moe_layout_offset(self.shape, L.LAYOUT_EXPERT_ROWS)
        self.expert_rows = self.layout[eo:eo + self.E_l]
        self.g_u_h = torch.empty((R, 3 * f), dtype=bf, device=dev)
        self.out = torch.empty((R, d), dtype=bf, device=dev)
        self.y = torch.empty((T, d), dtype=bf, device=dev)
        self.dgates = torch.empty((T, k), dtype=f32, device=dev)
        self.dlogits = torch.empty((T, E), dtype=f32, device=dev)
        self.dgu = torch.empty((R, 2 * f), dtype=bf, device=dev)
        self.dxr = torch.empty((R, d), dtype=bf, device=dev)
        self.dx_router = torch.empty((T, d), dtype=f32, device=dev)
        self.dx = torch.empty((T, d), dtype=bf, device=dev)
        self.dw_r = torch.empty((E, d), dtype=f32, device=dev)
        self._cur = 0       # which half of the double-buffered expert state is current
        self._states = {}   # name -> [buf0, buf1] symmetric [E_l, ...] (migratable state)
        if self.migratable:
            sy = self.ctx.symm_empty
            self._states["w_gu"] = [sy((self.E_l, 2 * f, d), bf) for _ in range(2)]
            self._states["w_down"] = [sy((self.E_l, d, f), bf) for _ in range(2)]
            self._states["dw_gu"] = [sy((self.E_l, 2 * f, d), f32) for _ in range(2)]
            self._states["dw_down"] = [sy((self.E_l, d, f), f32) for _ in range(2)]
            self.dw_gu = self._states["dw_gu"][0]
            self.dw_down = self._states["dw_down"][0]
        else:
            self.dw_gu = torch.empty((self.E_l, 2 * f, d), dtype=f32, device=dev)
            self.dw_down = torch.empty((self.E_l, d, f), dtype=f32, device=dev)
        if dims.ep_size > 1:
            self._verify_symmetric()
        self.rows_T = torch.tensor([T], dtype=i32, device=dev)
        self.fs = dims.E_shared * f
        if self.fs:
            fs = self.fs
            self.g_u_h_s = torch.empty((T, 3 * fs), dtype=bf, device=dev)
            self.y_s = torch.empty((T, d), dtype=bf, device=dev)
            self.dgu_s = torch.empty((T, 2 * fs), dtype=bf, device=dev)
            self.dx_s = torch.empty((T, d), dtype=bf, device=dev)
            self.dw_gu_s = torch.empty((1, 2 * fs, d), dtype=f32, device=dev)
            self.dw_down_s = torch.empty((1, d, fs), dtype=f32, device=dev)
        self.w_r = self.w_gu = self.w_down = self.bias = None
        self.w_gu_s = self.w_down_s = None
        # device memory this instance allocated (torch tensors + the ctx's allocations)
        self.torch_bytes = torch.cuda.memory_allocated(self.device) - torch_before

    # ------------------------------------------------------------------ weights
    def set_weights(self, w_r, w_gu, w_down, bias=None, w_gu_s=None, w_down_s=None):
        """w_r [E,d], w_gu [E_l,2f,d], w_down [E_l,d,f] (bf16, this rank's experts),
        bias [E] fp32 or None, shared w_gu_s [2fs,d], w_down_s [d,fs] or None."""
        dev = self.device
        self.w_r = w_r.to(dev, torch.bfloat16).contiguous()
        if self.migratable:
            self.w_gu = self._states["w_gu"][self._cur]
            self.w_down = self._states["w_down"][self._cur]
            self.w_gu.copy_(w_gu)
            self.w_down.copy_(w_down)
        else:
            self.w_gu = w_gu.to(dev, torch.bfloat16).contiguous()
            self.w_down = w_down.to(dev, torch.bfloat16).contiguous()
        self.bias = None if bias is None else bias.to(dev, torch.float32).contiguous()
        if self.fs:
            self.w_gu_s = w_gu_s.to(dev, torch.bfloat16).contiguous()
            self.w_down_s = w_down_s.to(dev, torch.bfloat16).contiguous()

    # ------------------------------------------------------------------ forward
    # EP = 1: moe_permute_dispatch_local (no send-layout copy, no transfer); False = the
    # general permute + dispatch path (tests compare the two)
    local_fast_path = True
    # NEXT-1 tile-granular overlap (fused path, no dedup): the dispatch runs inside the GEMM1
    # launch and every GEMM1 tile starts when its rows have arrived
    # (moe_dispatch_expert_ffn_up); False = moe_dispatch, then GEMM1.  None = auto: on when a
    # rank owns >= 8 experts -- GEMM1's first tiles wait for 1/E_l of the transfer (slot-major
    # order), so fine-grained layers gain (4-GPU box, profiles/r02/tile_overlap: DS-MoE N=4
    # 1.80 vs 1.84 ms, V3-like N=4 25.6-26.5 vs 26.5 ms) and coarse ones lose (Mixtral N=4,
    # E_l = 2: 3.59-3.60 vs 3.52-3.55 ms).  MOE_TILE_OVERLAP=0/1 forces it.
    tile_overlap = {"0": False, "1": True}.get(os.environ.get("MOE_TILE_OVERLAP", ""))
    tile_overlap_min_experts = 8
    # the backward twin (combine_bwd inside dgrad-1) with tile_overlap.  None = auto: only
    # without shared experts -- with them the separate combine_bwd runs beside the shared-expert
    # backward GEMMs, which the fused launch would serialise (4-GPU box,
    # profiles/r02/tile_overlap/run4: DS-MoE N=4 2.03 ms fwd+bwd fused vs 1.80 forward only vs
    # 1.84 off; V3-like N=4 25.6-25.8 vs 26.9 off).  MOE_TILE_OVERLAP_BWD=0/1 forces it.
    tile_overlap_bwd = {"0": False, "1": True}.get(os.environ.get("MOE_TILE_OVERLAP_BWD", ""))

    def _tile_overlap_bwd(self) -> bool:
        on = self.tile_overlap_bwd
        if on is None:
            on = not self.fs
        return bool(on) and self._tile_overlap()
    # per-phase CUDA-event markers (bench.py --breakdown); off by default
    marks = None
    # SMs given to an all-to-all that runs beside a GEMM (the GEMM gets the rest).  Measured on
    # DS-MoE N=4 (profiles/r01/sms_*.json): 20 -> 1.97 ms, 48 -> 1.92 ms (dedup 2.01 -> 1.89),
    # 74 -> 2.00 ms (dedup)
    comm_sms = 48
    # SM budget of every all-to-all outside the overlap (0 = all SMs); the PP x EP executor
    # leaves a few SMs free so the NCCL stage-to-stage kernels can always be scheduled beside
    # a spinning collective
    base_comm_sms = 0

    def set_base_comm_sms(self, n):
        self.base_comm_sms = int(n)
        self.ctx.set_sm_limits(0, self.base_comm_sms)

    def _concurrent(self, comm_fn, gemm_fn):
        """comm_fn(stream) on a side stream with `comm_sms` SMs, gemm_fn(stream) on the current
        stream with the remaining SMs; both ordered after everything issued so far, and the
        current stream waits for both at the end."""
        main = torch.cuda.current_stream(self.device)
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        side = self._side
        start = torch.cuda.Event()
        start.record(main)
        side.wait_event(start)
        n_sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        # GEMM first: its CTAs (one per SM, ~213 KB smem) take their SMs, the transfer blocks
        # fill the SMs left over
        self.ctx.set_sm_limits(n_sms - self.comm_sms, 0)
        gemm_fn(main)
        self.ctx.set_sm_limits(0, self.comm_sms)
        comm_fn(side)
        self.ctx.set_sm_limits(0, self.base_comm_sms)
        done = torch.cuda.Event()
        done.record(side)
        main.wait_event(done)

    def _mark(self, name):
        if self.marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.marks.append((name, ev))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x [T_local, d] bf16 on this rank's device -> y [T_local, d] bf16."""
        c = self.ctx
        self.x = x
        f, T = self.dims.f, self.dims.T_local
        self._mark("start")
        L.moe_router_logits(c, x, self.w_r, self.bias, self.logits)
        L.moe_route(c, self.logits, self.topk_idx, self.gates)
        self._mark("F0+F1 router,route")
        if self.dedup:
            return self._forward_dedup(x)
        if self.dims.ep_size == 1 and self.local_fast_path:
            # EP = 1 is local only: the permute writes the receive layout directly
            L.moe_permute_dispatch_local(c, x, self.topk_idx, self.counts, self.dest_row,
                                         self.layout, self.xr)
            self._mark("F2+F3 permute (local)")
            y_extra = None
            if self.fs:
                L.moe_expert_ffn(c, x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s,
                                 self.g_u_h_s, self.y_s)
                y_extra = self.y_s
                self._mark("F4s shared ffn")
            # dest_row now holds receive rows: the GEMMs write the receive layout with plain
            # TMA-store epilogues and F6 gathers O in place (no send-layout copy, no flags)
            L.moe_expert_ffn(c, self.xr, self.expert_rows, self.E_l, self.R, f, self.w_gu,
                             self.w_down, self.g_u_h, self.out)
            self._mark("F4 expert ffn")
            L.moe_unpermute(c, self.out, self.gates, self.dest_row, y_extra, self.y)
            self._mark("F6 unpermute")
            return self.y
        L.moe_permute(c, x, self.topk_idx, self.counts, self.dest_row, self.xs)
        self._mark("F2 permute")
        y_extra = None
        if self._tile_overlap():
            # F3 + F4 up in one launch: GEMM1 tiles start as their rows land (NEXT-1)
            L.moe_dispatch_expert_ffn_up(c, self.xs, self.counts, self.layout, self.xr, self.w_gu,
                                         self.g_u_h)
            self._mark("F3+F4 dispatch + GEMM1 (tile-granular overlap)")
            if self.fs:
                L.moe_expert_ffn(c, x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s,
                                 self.g_u_h_s, self.y_s)
                y_extra = self.y_s
                self._mark("F4s shared ffn")
            L.moe_expert_ffn_down_combine(c, self.layout, self.w_down, self.g_u_h, self.ys,
                                          self.gates, self.dest_row, y_extra, self.y)
            self._mark("F4+F5+F6 GEMM2 + combine")
            return self.y
        if self.fs and self.overlap:
            # shared experts (local tokens, no exchange) run beside the dispatch all-to-all on
            # disjoint SMs: dispatch on a side stream, shared GEMMs on this one
            self._concurrent(lambda s: L.moe_dispatch(c, self.xs, self.counts, self.layout,
                                                      self.xr, stream=s),
                             lambda s: L.moe_expert_ffn(c, x, self.rows_T, 1, T, self.fs,
                                                        self.w_gu_s, self.w_down_s, self.g_u_h_s,
                                                        self.y_s, stream=s))
            y_extra = self.y_s
            self._mark("F3 dispatch || F4s shared ffn")
        else:
            L.moe_dispatch(c, self.xs, self.counts, self.layout, self.xr)
            self._mark("F3 dispatch")
            if self.fs:
                L.moe_expert_ffn(c, x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s,
                                 self.g_u_h_s, self.y_s)
                y_extra = self.y_s
                self._mark("F4s shared ffn")
        return self._forward_reverse(y_extra)

    def _forward_reverse(self, y_extra):
        """F4 + the per-slot combine (fused into GEMM2's epilogue unless stepwise) + F6."""
        c, f = self.ctx, self.dims.f
        if self.fused:
            # GEMM2's epilogue stores O rows straight into the sources' ys (combine fused)
            L.moe_expert_ffn_combine(c, self.xr, self.layout, self.w_gu, self.w_down, self.g_u_h,
                                     self.ys, self.gates, self.dest_row, y_extra, self.y)
            self._mark("F4+F5+F6 expert ffn + combine")
        else:
            L.moe_expert_ffn(c, self.xr, self.expert_rows, self.E_l, self.R, f, self.w_gu,
                             self.w_down, self.g_u_h, self.out)
            self._mark("F4 expert ffn")
            L.moe_combine(c, self.out, self.layout, self.ys, self.gates, self.dest_row, y_extra,
                          self.y)
            self._mark("F5+F6 combine")
        return self.y

    # ------------------------------------------------------------------ NEXT-4 dedup all-to-all
    def _forward_dedup(self, x):
        c, T, f = self.ctx, self.dims.T_local, self.dims.f
        L.moe_permute(c, x, self.topk_idx, self.counts, self.dest_row, None)
        L.moe_dedup_pairs(c, self.topk_idx, self.dest_row, self.pdest, self.ntok)
        self._mark("F2 permute (indices) + pairs")

        def dispatch(s):
            L.moe_dedup_dispatch(c, x, self.counts, self.ntok, self.pdest, self.dest_row,
                                 self.topk_idx, self.gates, self.layout, self.dlayout, self.xt,
                                 self.rlist, self.glist, self.xr, stream=s)
        y_extra = None
        if self.fs and self.overlap:
            self._concurrent(dispatch, lambda s: L.moe_expert_ffn(
                c, x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s, self.g_u_h_s,
                self.y_s, stream=s))
            y_extra = self.y_s
        else:
            dispatch(None)
            if self.fs:
                L.moe_expert_ffn(c, x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s,
                                 self.g_u_h_s, self.y_s)
                y_extra = self.y_s
        self._mark("F3 dedup dispatch + expand")
        if self.dedup_mode == "dispatch":
            return self._forward_reverse(y_extra)
        L.moe_expert_ffn(c, self.xr, self.expert_rows, self.E_l, self.R, f, self.w_gu, self.w_down,
                         self.g_u_h, self.out)
        self._mark("F4 expert ffn")
        L.moe_dedup_combine(c, self.out, self.dlayout, self.rlist, self.glist, self.pdest, y_extra,
                            self.ys, self.y)
        self._mark("F5+F6 dedup combine")
        return self.y

    def _backward_dedup(self, dy, accumulate):
        c, T, f = self.ctx, self.dims.T_local, self.dims.f

        def combine_bwd(s):
            if self.dedup_mode == "dispatch":   # O rows are in ys (fused GEMM2 stores)
                L.moe_dedup_combine_bwd_ys(c, dy, self.gates, self.dest_row, self.ys, self.pdest,
                                           self.layout, self.dlayout, self.rlist, self.glist,
                                           self.xt, self.dgates, self.dout_r, stream=s)
            else:
                L.moe_dedup_combine_bwd(c, dy, self.pdest, self.layout, self.dlayout, self.rlist,
                                        self.glist, self.out, self.xt, self.dg_own, self.dout_r,
                                        stream=s)
        shared_done = False
        if self.fs and self.overlap:
            self._concurrent(combine_bwd, lambda s: L.moe_expert_ffn_bwd(
                c, self.x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s, self.g_u_h_s,
                dy, self.dgu_s, self.dx_s, self.dw_gu_s, self.dw_down_s, accumulate, stream=s))
            shared_done = True
        else:
            combine_bwd(None)
        self._mark("B6+B5 dedup combine_bwd")
        if self.dedup_mode == "dispatch":
            return self._backward_reverse(dy, accumulate, shared_done)
        L.moe_expert_ffn_bwd(c, self.xr, self.expert_rows, self.E_l, self.R, f, self.w_gu,
                             self.w_down, self.g_u_h, self.dout_r, self.dgu, self.dxr, self.dw_gu,
                             self.dw_down, accumulate)
        self._mark("B4 expert ffn_bwd")
        L.moe_dedup_dispatch_bwd(c, self.dxr, self.dlayout, self.rlist, self.dg_own, self.pdest,
                                 self.dest_row, self.topk_idx, self.dxs, self.dgpart, self.dgates)
        self._mark("B3 dedup dispatch_bwd")
        return self._backward_tail(dy, accumulate, shared_done)

    # ------------------------------------------------------------------ backward
    def backward(self, dy: torch.Tensor, accumulate: bool = False) -> torch.Tensor:
        """dy [T_local, d] bf16 -> dx [T_local, d] bf16; fills dw_r, dw_gu, dw_down
        (and dw_gu_s, dw_down_s) as fp32 per-rank gradients."""
        c = self.ctx
        f, T = self.dims.f, self.dims.T_local
        if self.dedup:
            return self._backward_dedup(dy, accumulate)
        if self.dims.ep_size == 1 and self.local_fast_path:
            # receive layout in place (moe_permute_dispatch_local): dO = g dy and dgates on the
            # expert outputs, the FFN backward writes dX rows to dxr, the gathers read them there
            L.moe_combine_bwd_local(c, dy, self.gates, self.dest_row, self.out, self.layout,
                                    self.dgates, self.dout_r)
            self._mark("B6 combine_bwd (local)")
            L.moe_expert_ffn_bwd(c, self.xr, self.expert_rows, self.E_l, self.R, f, self.w_gu,
                                 self.w_down, self.g_u_h, self.dout_r, self.dgu, self.dxr,
                                 self.dw_gu, self.dw_down, accumulate)
            self._mark("B4 expert ffn_bwd")
            return self._backward_tail(dy, accumulate, False, rows=self.dxr)
        if self._tile_overlap_bwd():
            # B6+B5 + dgrad-1 in one launch: dO tiles start as their rows land (NEXT-1)
            L.moe_combine_bwd_expert_ffn_dh(c, dy, self.gates, self.dest_row, self.ys, self.layout,
                                            self.dgates, self.dout_r, self.w_down, self.g_u_h,
                                            self.dgu)
            self._mark("B6+B5+B4 combine_bwd + dgrad-1 (tile-granular overlap)")
            L.moe_expert_ffn_bwd_dx_dispatch(c, self.xr, self.layout, self.w_gu, self.g_u_h,
                                             self.dout_r, self.dgu, self.dxs, self.dw_gu,
                                             self.dw_down, accumulate)
            self._mark("B4+B3 dgrad-2 + wgrads + dispatch_bwd")
            return self._backward_tail(dy, accumulate, False)
        shared_done = False
        if self.fs and self.overlap:
            # shared-expert backward (needs only dy) beside the combine_bwd all-to-all
            self._concurrent(lambda s: L.moe_combine_bwd(c, dy, self.gates, self.dest_row, self.ys,
                                                         self.layout, self.dgates, self.dout_r,
                                                         stream=s),
                             lambda s: L.moe_expert_ffn_bwd(c, self.x, self.rows_T, 1, T, self.fs,
                                                            self.w_gu_s, self.w_down_s,
                                                            self.g_u_h_s, dy, self.dgu_s,
                                                            self.dx_s, self.dw_gu_s,
                                                            self.dw_down_s, accumulate, stream=s))
            shared_done = True
            self._mark("B6+B5 combine_bwd || B4s shared ffn_bwd")
        else:
            L.moe_combine_bwd(c, dy, self.gates, self.dest_row, self.ys, self.layout, self.dgates,
                              self.dout_r)
            self._mark("B6+B5 combine_bwd")
        return self._backward_reverse(dy, accumulate, shared_done)

    def _backward_reverse(self, dy, accumulate, shared_done):
        """B4 + the per-slot dispatch_bwd (fused into dgrad-2's epilogue unless stepwise)."""
        c, f = self.ctx, self.dims.f
        if self.fused:
            # dgrad-2's epilogue stores dX rows straight into the sources' dxs; the wgrad
            # GEMMs run while those stores drain
            L.moe_expert_ffn_bwd_dispatch(c, self.xr, self.layout, self.w_gu, self.w_down,
                                          self.g_u_h, self.dout_r, self.dgu, self.dxs, self.dw_gu,
                                          self.dw_down, accumulate)
            self._mark("B4+B3 expert ffn_bwd + dispatch_bwd")
        else:
            L.moe_expert_ffn_bwd(c, self.xr, self.expert_rows, self.E_l, self.R, f, self.w_gu,
                                 self.w_down, self.g_u_h, self.dout_r, self.dgu, self.dxr,
                                 self.dw_gu, self.dw_down, accumulate)
            self._mark("B4 expert ffn_bwd")
            L.moe_dispatch_bwd(c, self.dxr, self.layout, self.dxs)
            self._mark("B3 dispatch_bwd")
        return self._backward_tail(dy, accumulate, shared_done)

    def _backward_tail(self, dy, accumulate, shared_done, rows=None):
        """Shared experts (if not yet done), route / router backward and permute backward
        (gathering dX rows from `rows`: dxs, or dxr on the EP = 1 receive layout)."""
        rows = self.dxs if rows is None else rows
        c, T = self.ctx, self.dims.T_local
        dx_extra = self.dx_s if self.fs else None
        if self.fs and not shared_done:
            L.moe_expert_ffn_bwd(c, self.x, self.rows_T, 1, T, self.fs, self.w_gu_s, self.w_down_s,
                                 self.g_u_h_s, dy, self.dgu_s, self.dx_s, self.dw_gu_s,
                                 self.dw_down_s, accumulate)
            self._mark("B4s shared ffn_bwd")
        L.moe_route_bwd(c, self.logits, self.topk_idx, self.gates, self.dgates, self.dlogits)
        if self.dims.k > 1:
            # dl is k-sparse: dx_router is gathered inside the permute backward (exact fp32)
            L.moe_router_logits_bwd(c, self.x, self.w_r, self.dlogits, None, self.dw_r, accumulate)
            self._mark("B1+B0 route_bwd,router dW")
            if self.dedup_mode == "all":   # dxs holds the pair partials, rows pdest [T, EP]
                L.moe_dedup_permute_bwd_router(c, self.dxs, self.pdest, self.topk_idx,
                                               self.dlogits, self.w_r, dx_extra, self.dx)
            else:
                L.moe_permute_bwd_router(c, rows, self.dest_row, self.topk_idx, self.dlogits,
                                         self.w_r, dx_extra, self.dx)
        else:
            L.moe_router_logits_bwd(c, self.x, self.w_r, self.dlogits, self.dx_router, self.dw_r,
                                    accumulate)
            self._mark("B1+B0 route_bwd,router dW")
            L.moe_permute_bwd(c, rows, self.dest_row, self.dx_router, dx_extra, self.dx)
        self._mark("B2 permute_bwd")
        return self.dx

    # ------------------------------------------------------------------ CUDA graph
    def capture(self, x: torch.Tensor, dy: torch.Tensor, accumulate: bool = False, post=None):
        """Records forward(x) + backward(dy) (+ post(), e.g. copies of self.y / self.dx) into a
        CUDA graph and returns it; graph.replay() reruns the step on the CURRENT contents of x
        and dy.  The collectives' epoch lives on the device (it is advanced by the kernels, not
        baked into their arguments), so every replay is a fresh exchange.  All ranks of the EP
        group must capture (one eager warm-up step, then the capture) and replay in lockstep.
        Placement changes (migrate) invalidate the graph: capture again afterwards."""
        dev = self.device
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            self.forward(x)
            self.backward(dy, accumulate)
            if post is not None:
                post()
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.forward(x)
            self.backward(dy, accumulate)
            if post is not None:
                post()
        return g

    # ------------------------------------------------------------------ expert migration
    # SURVEY.md §8(f) NEXT-2 / PAPER.md §VI: the router "maintains token distribution"
    # (PAPER.md:648); Alg. 2 rebalances; experts move with their weights.

    def observe_loads(self):
        """Adds this call's routed rows per expert (from the layout record, identical on every
        rank) to the running load histogram.  One small device->host copy (a sync point)."""
        EP, E = self.dims.ep_size, self.dims.E
        cm = self.layout[:EP * E].view(EP, E).sum(0).to(torch.int64).cpu()
        self.loads = cm if getattr(self, "loads", None) is None else self.loads + cm
        return self.loads

    def rebalance(self, loads=None, max_iters=100, group=None):
        """Runs Alg. 2 (libmoe moe_rebalance) on the load histogram and migrates the experts
        that moved.  Every rank computes the same placement from the same loads, so no extra
        agreement step is needed.  Returns (swap count, experts moved)."""
        loads = self.loads if loads is None else loads
        new, swaps = L.moe_rebalance([int(v) for v in loads], self.dims.ep_size, self.placement,
                                     max_iters)
        moved = self.migrate(new, group)
        self.loads = None
        return swaps, moved

    # imbalance threshold of maybe_rebalance (reading R20): the most-loaded EP rank receives
    # more than 10 % above the mean
    rebalance_threshold = 1.10

    def memory_account(self):
        """Device bytes held by this layer instance (measured: torch allocations made by the
        constructor + every allocation of the libmoe ctx) and the part that is the saved expert
        activations Eq. 4 counts per token-slot as 3 d_ffn + d_model (reading
        R9): xr [R, d] and g_u_h [R, 3f] for R = moe_recv_rows_max receive rows."""
        heap, used, ctx_total = self.ctx.device_bytes()
        saved = self.xr.numel() * 2 + self.g_u_h.numel() * 2
        return {"torch_bytes": int(self.torch_bytes), "ctx_bytes": int(ctx_total),
                "total_bytes": int(self.torch_bytes + ctx_total), "heap_bytes": int(heap),
                "saved_expert_activation_bytes": int(saved), "recv_rows": int(self.R)}

    def imbalance(self, loads=None):
        """max / mean of the EP ranks' routed rows over the observed loads (libmoe)."""
        loads = self.loads if loads is None else loads
        return L.moe_load_imbalance([int(v) for v in loads], self.placement, self.dims.ep_size)

    def maybe_rebalance(self, threshold=None, max_iters=100):
        """The external scheduler of PAPER.md:648: when the observed imbalance crosses the
        threshold, run Alg. 2 and migrate; otherwise keep accumulating loads.  Every rank
        sees the same loads (the layout record), so every rank takes the same decision.
        Returns (imbalance, swaps, experts moved) -- swaps = moved = 0 if below."""
        if self.loads is None or self.dims.ep_size == 1:
            return 1.0, 0, 0
        thr = self.rebalance_threshold if threshold is None else threshold
        imb = self.imbalance()
        if imb <= thr:
            return imb, 0, 0
        swaps, moved = self.rebalance(max_iters=max_iters)
        return imb, swaps, moved

    def _verify_symmetric(self):
        """Every rank must have made the same symmetric allocations (peers write at OUR
        offsets): compare the allocation fingerprints (moe_ctx_verify_symmetric)."""
        self.ctx.verify_symmetric(_all_gather_bytes(self.ctx.fingerprint(), self.group))

    def expert_state(self, name, per_expert_shape, dtype):
        """Registers per-expert state [E_l, *per_expert_shape] (e.g. optimizer moments) that
        migrate() moves with the experts; returns the current buffer.  Collective (symmetric
        allocation); needs migratable=True and expert_state_bytes room."""
        if not self.migratable:
            raise RuntimeError("expert_state needs MoELayer(migratable=True)")
        shape = (self.E_l, *per_expert_shape)
        self._states[name] = [self.ctx.symm_empty(shape, dtype) for _ in range(2)]
        if self.dims.ep_size > 1:
            self._verify_symmetric()
        return self._states[name][self._cur]

    def state(self, name):
        """Current buffer of a migratable per-expert state ("w_gu", "w_down", "dw_gu",
        "dw_down" or a registered name)."""
        return self._states[name][self._cur]

    def migrate(self, new_placement, group=None):
        """Moves every expert's state (bf16 weights, fp32 weight gradients and any state
        registered with expert_state) to the owners given by new_placement (expert -> global
        slot) and switches the ctx to it.  Collective over the EP group.  Each tensor moves
        with ONE moe_migrate launch: old owners push their experts straight into the new
        owners' other half of the double buffer over the peer maps (PAPER.md:648's migration
        of experts with their state -- 48 d f bytes each incl. optimizer state, Table
        PAPER.md:650-668).  Gradients move WITH their experts, so an accumulation in progress
        stays credited to the right expert.  Invalidates captured CUDA graphs.  Returns the
        number of experts that changed rank."""
        E_l, r = self.E_l, self.dims.ep_rank
        old = list(self.placement)
        new = [int(v) for v in new_placement]
        if sorted(new) != list(range(self.dims.E)):
            raise ValueError("new_placement must be a permutation of range(E)")
        moved = sum(1 for e in range(self.dims.E) if old[e] // E_l != new[e] // E_l)
        if self.migratable:
            nxt = 1 - self._cur
            for bufs in self._states.values():
                L.moe_migrate(self.ctx, old, new, bufs[self._cur], bufs[nxt])
            self._cur = nxt
            self.w_gu, self.w_down = self._states["w_gu"][nxt], self._states["w_down"][nxt]
            self.dw_gu, self.dw_down = self._states["dw_gu"][nxt], self._states["dw_down"][nxt]
        else:
            if moved:
                raise RuntimeError("moving experts between ranks needs MoELayer(migratable=True)")
            # local slot permutation (EP = 1 or an intra-rank reshuffle)
            perm = torch.empty(E_l, dtype=torch.int64)
            for e in range(self.dims.E):
                if new[e] // E_l == r:
                    perm[new[e] % E_l] = old[e] % E_l
            perm = perm.to(self.device)
            self.w_gu = self.w_gu.index_select(0, perm).contiguous()
            self.w_down = self.w_down.index_select(0, perm).contiguous()
            self.dw_gu.copy_(self.dw_gu.index_select(0, perm))
            self.dw_down.copy_(self.dw_down.index_select(0, perm))
        self.placement = new
        self.ctx.set_placement(new)
        return moved

    def experts_of_slots(self):
        """Global expert id held in each local slot of this rank."""
        inv = [0] * self.dims.E
        for e, s in enumerate(self.placement):
            inv[s] = e
        r, E_l = self.dims.ep_rank, self.E_l
        return inv[r * E_l:(r + 1) * E_l]

    def _tile_overlap(self) -> bool:
        # (EP = 1 reaches the general path only with local_fast_path = False, i.e. in tests)
        on = self.tile_overlap
        if on is None:
            on = self.E_l >= self.tile_overlap_min_experts
        return bool(on) and self.fused and not self.dedup

    def kernel_launches(self, fwd=True, bwd=True) -> int:
        """Number of libmoe kernels one forward / backward launches (for bench.py)."""
        n = 0
        if self.dedup:
            # fwd: router GEMM, route, permute (2, no scatter), pairs (2), dispatch (transfer +
            # expand), ffn (2), combine (reduce + gather | fused: wait + gather); bwd:
            # combine_bwd (transfer + expand), ffn_bwd (4 | fused: 4 + wait), dispatch_bwd
            # (reduce + dgates | fused: none), route_bwd, router bwd (3), permute_bwd
            rev = self.dedup_mode == "dispatch" and self.fused
            if fwd:
                n += 1 + 1 + 2 + 2 + 2 + 2 + 2 + (2 if self.fs else 0)
            if bwd:
                n += 2 + 4 + (1 if rev else 2) + 1 + 3 + 1 + (4 if self.fs else 0)
            return n
        if self.dims.ep_size == 1 and self.local_fast_path:
            # receive layout in place: fwd router GEMM, route, permute (3), ffn (2), unpermute;
            # bwd combine_bwd_local, ffn_bwd (4), route_bwd, router bwd (3, +2 for k = 1),
            # permute_bwd
            if fwd:
                n += 1 + 1 + 3 + 2 + 1 + (2 if self.fs else 0)
            if bwd:
                n += 1 + 4 + 1 + 3 + (0 if self.dims.k > 1 else 2) + 1 + (4 if self.fs else 0)
            return n
        if fwd:
            # router GEMM, route, permute (3), dispatch (1 fused launch), ffn (2), combine (2)
            n += 1 + 1 + 3 + 1 + 2 + 2 + (2 if self.fs else 0)
            if self._tile_overlap():
                n -= 1   # dispatch + GEMM1 are one launch
        if bwd:
            # combine_bwd (1), ffn_bwd (4), dispatch_bwd (1), route_bwd,
            # router bwd (hi/lo split, split-K dW_r GEMM, partial sum; k = 1 adds the
            # stacked-W_r copy and the dense dgrad GEMM), permute_bwd
            n += 1 + 4 + 1 + 1 + 3 + (0 if self.dims.k > 1 else 2) + 1 + (4 if self.fs else 0)
            if self._tile_overlap_bwd():
                n -= 1   # combine_bwd + dgrad-1 are one launch
        return n

    def close(self):
        self.ctx.close()

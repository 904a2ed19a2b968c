"""PP x EP pipelined executor of a stack of MoE layers.

PAPER.md:149: the P GPUs form a PP x EP mesh -- PP pipeline stages, each staffed by EP GPUs
that hold L/PP layers and E/EP experts per layer (expert-data parallelism inside the stage,
PAPER.md:272); stage i's EP GPU e sends its activations to "its counterpart" (i+1, e)
 and receives gradients back.  Micro-batches run in the 1F1B order of libmoe's
moe_pipeline_1f1b (reading R19), so stage i holds at most PP - i
micro-batches in flight: each layer keeps that many activation contexts (MoELayer instances
sharing the layer's weights and accumulating into one set of weight gradients).

Mesh: global rank = stage * EP + e (EP groups contiguous, "EP within the fast
domain").  Stage-to-stage transfers use torch.distributed point-to-point (NCCL), the plumbing;
every step of every layer runs through libmoe.  Activations leave through a per-micro-batch
send buffer, so a layer's output buffer can be reused while the transfer is still queued.
"""
from __future__ import annotations

import torch

from . import _lib as L
from .layer import LayerDims, MoELayer


class PipelineStack:
    def __init__(self, dims: LayerDims, n_layers: int, pp: int, n_micro: int, device=0,
                 fused: bool = True, dedup=False, free_sms: int = 8, layer_cls=MoELayer):
        """dims: one layer's shape for ONE micro-batch on this EP rank (T_local = tokens of the
        micro-batch / EP, ep_size = EP, ep_rank = this rank's index in its stage).  Collective
        over the whole world (every rank builds its stage's EP group).  layer_cls / device=None
        exist for the CPU (gloo) test of the schedule and the stage-to-stage routing."""
        import torch.distributed as dist
        self.dist = dist
        world, rank = dist.get_world_size(), dist.get_rank()
        ep = dims.ep_size
        if world != pp * ep or n_layers % pp:
            raise ValueError(f"need world == PP x EP and PP | L (world {world}, PP {pp}, EP {ep}, "
                             f"L {n_layers})")
        self.pp, self.ep, self.M = pp, ep, n_micro
        self.stage, self.e = divmod(rank, ep)
        if dims.ep_rank != self.e:
            raise ValueError("dims.ep_rank must be this rank's index in its stage")
        self.device = torch.device("cpu" if device is None else f"cuda:{device}")
        groups = [dist.new_group(list(range(i * ep, (i + 1) * ep))) for i in range(pp)]
        self.group = groups[self.stage]
        self.prev = (self.stage - 1) * ep + self.e if self.stage > 0 else None
        self.next = (self.stage + 1) * ep + self.e if self.stage < pp - 1 else None
        self.ops = L.moe_pipeline_1f1b(pp, self.stage, n_micro)
        self.n_slots = min(pp - self.stage, n_micro)       # PAPER.md:284 in-flight bound
        self.n_local = n_layers // pp
        n_sms = (torch.cuda.get_device_properties(self.device).multi_processor_count
                 if device is not None else 0)
        self.layers = []                                    # [local layer][slot]
        for _ in range(self.n_local):
            # slot 0 owns the layer's (migratable) expert state; the other activation contexts
            # share it by reference (set_weights), so they need no state buffers of their own
            slots = [layer_cls(dims, device=device, group=self.group, fused=fused, dedup=dedup,
                               migratable=None if i == 0 else False)
                     for i in range(self.n_slots)]
            if n_sms:
                for s in slots:
                    s.set_base_comm_sms(n_sms - free_sms)
            self.layers.append(slots)
        T, d = dims.T_local, dims.d
        bf = torch.bfloat16
        buf = lambda: [torch.empty((T, d), dtype=bf, device=self.device) for _ in range(n_micro)]
        # separate buffers per direction: a received activation stays the first layer's saved
        # input until the micro-batch's backward, while its gradient arrives in another buffer
        self.send_act, self.send_grad = buf(), buf()
        self.recv_act, self.recv_grad = buf(), buf()
        self.y_out, self.dx_out = buf(), buf()
        self.record = None   # tests: {(local layer, m): {...}} clones of each layer's tensors

    # ------------------------------------------------------------------ weights
    def set_weights(self, l, w_r, w_gu, w_down, bias=None, w_gu_s=None, w_down_s=None):
        """Local layer l (global layer stage * L/PP + l): every activation context shares the
        weights and the weight-gradient buffers."""
        slots = self.layers[l]
        for s in slots:
            s.set_weights(w_r, w_gu, w_down, bias, w_gu_s, w_down_s)
        self._share(l)

    def _share(self, l):
        s0 = self.layers[l][0]
        for s in self.layers[l][1:]:
            s.w_r, s.w_gu, s.w_down, s.bias = s0.w_r, s0.w_gu, s0.w_down, s0.bias
            s.w_gu_s, s.w_down_s = s0.w_gu_s, s0.w_down_s
            s.dw_r, s.dw_gu, s.dw_down = s0.dw_r, s0.dw_gu, s0.dw_down
            if s0.fs:
                s.dw_gu_s, s.dw_down_s = s0.dw_gu_s, s0.dw_down_s

    def migrate(self, l, new_placement):
        """Expert migration of local layer l as ONE stack-level operation: slot 0 moves the
        layer's expert state (weights and gradients, MoELayer.migrate), every other activation
        context is re-pointed at the moved tensors and switched to the new placement.
        Collective over the stage's EP group; call between steps."""
        slots = self.layers[l]
        moved = slots[0].migrate(new_placement)
        for s in slots[1:]:
            s.placement = list(slots[0].placement)
            s.ctx.set_placement(s.placement)
        self._share(l)
        return moved

    def memory_report(self):
        """Per-stage device memory of this rank against PAPER.md Eq. 4 (1F1B, stage i holds
        PP - i in-flight micro-batches): for every local layer the number of
        activation contexts, the measured bytes of each (MoELayer.memory_account), and Eq. 4's
        expert-activation term for one micro-batch on this rank, 2 (b/M) s k / EP (3 d_ffn +
        d_model) bytes = 2 T_local k (3 f + d) (reading R19: the attention terms do not exist
        in an MoE-only stack)."""
        d0 = self.layers[0][0].dims
        eq4_term = 2 * d0.T_local * d0.k * (3 * d0.f + d0.d)
        layers = []
        for slots in self.layers:
            acc = [s.memory_account() for s in slots]
            layers.append({"n_slots": len(slots),
                           "slot_total_bytes": [a["total_bytes"] for a in acc],
                           "saved_expert_activation_bytes": [a["saved_expert_activation_bytes"]
                                                             for a in acc]})
        return {"stage": self.stage, "pp": self.pp, "in_flight_bound": min(self.pp - self.stage,
                                                                            self.M),
                "eq4_expert_activation_bytes_per_microbatch": eq4_term,
                "stage_bytes": sum(sum(l["slot_total_bytes"]) for l in layers),
                "layers": layers}

    def grads(self, l):
        s0 = self.layers[l][0]
        return s0.dw_r, s0.dw_gu, s0.dw_down

    # ------------------------------------------------------------------ one step
    def step(self, xs=None, dys=None):
        """One training step over the M micro-batches in 1F1B order.  Stage 0 passes xs (M
        tensors [T_local, d] bf16), the last stage dys (the upstream gradients of its outputs).
        Returns (ys, dxs): the last stage's outputs and stage 0's input gradients (lists of M
        tensors, valid until the next step), None elsewhere.  Weight gradients of the step are
        in grads(l) (the first backward overwrites, the others accumulate)."""
        dist = self.dist
        pending = []
        last = self.next is None
        for kind, m in self.ops:
            slot = m % self.n_slots
            if kind == L.PIPE_FORWARD:
                if self.prev is None:
                    h = xs[m]
                else:
                    self._recv(self.recv_act[m], self.prev)
                    h = self.recv_act[m]
                for l in range(self.n_local):
                    lay = self.layers[l][slot]
                    x_in = h
                    h = lay.forward(h)
                    if self.record is not None:
                        self._rec(l, m, x=x_in, y=h, logits=lay.logits, topk=lay.topk_idx,
                                  dest=lay.dest_row)
                if last:
                    self.y_out[m].copy_(h)
                else:
                    self.send_act[m].copy_(h)
                    pending.append(self._send(self.send_act[m], self.next))
            else:
                if last:
                    g = dys[m]
                else:
                    self._recv(self.recv_grad[m], self.next)
                    g = self.recv_grad[m]
                for l in reversed(range(self.n_local)):
                    lay = self.layers[l][slot]
                    dy_in = g
                    g = lay.backward(g, accumulate=m > 0)
                    if self.record is not None:
                        self._rec(l, m, dy=dy_in, dx=g)
                if self.prev is None:
                    self.dx_out[m].copy_(g)
                else:
                    self.send_grad[m].copy_(g)
                    pending.append(self._send(self.send_grad[m], self.prev))
        for p in pending:
            p.wait()
        return (self.y_out if last else None), (self.dx_out if self.prev is None else None)

    def _host_staged(self):
        """gloo moves CPU tensors only: with a gloo group and device tensors (several ranks
        sharing one GPU in the tests, tests/mp_common.py) the hand-offs go through host
        copies; NCCL (one GPU per rank) moves device memory directly."""
        return self.device.type == "cuda" and self.dist.get_backend() == "gloo"

    def _send(self, buf, dst):
        if self._host_staged():
            return self.dist.isend(buf.cpu(), dst=dst)   # .cpu() waits for the producer
        return self.dist.isend(buf, dst=dst)

    def _recv(self, buf, src):
        if self._host_staged():
            h = torch.empty(buf.shape, dtype=buf.dtype)
            self.dist.recv(h, src=src)
            buf.copy_(h)
        else:
            self.dist.irecv(buf, src=src).wait()

    def capture(self, xs=None, dys=None):
        """Records one step(xs, dys) -- every layer call and the NCCL stage hand-offs -- into a
        CUDA graph and returns it; graph.replay() reruns the step on the current contents of
        xs / dys (outputs in the buffers step() returns).  Collective: every rank captures
        (one eager warm-up step on the capture stream first) and replays in lockstep."""
        if self._host_staged():
            raise RuntimeError("CUDA-graph capture needs device-side (NCCL) stage hand-offs")
        dev = self.device
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            self.step(xs, dys)
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        self.dist.barrier()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.step(xs, dys)
        torch.cuda.synchronize(dev)
        self.dist.barrier()
        return g

    def _rec(self, l, m, **tensors):
        r = self.record.setdefault((l, m), {})
        for k, t in tensors.items():
            r[k] = t.detach().clone()

    def close(self):
        for slots in self.layers:
            for s in slots:
                s.close()

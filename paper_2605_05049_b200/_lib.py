"""ctypes binding of libmoe.so (include/moe.h) -- argument marshalling only.

Every function here has the name of the C entry point it calls, takes torch
tensors (device memory owned by the caller) and passes their raw pointers and
the current CUDA stream.  No step of the layer is computed in Python.  If the
library is missing the import fails loudly: there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# MOE_LIB: an instrumented in-tree build of the same sources (tools/trace_a2a.py)
LIB_PATH = os.environ.get("MOE_LIB") or os.path.join(_HERE, "libmoe.so")

MOE_ALIGN_ROWS = 128
MOE_IPC_HANDLE_BYTES = 64
LAYOUT_COUNTS_ALL, LAYOUT_EXPERT_ROWS, LAYOUT_SEG_BASE = 0, 1, 2

_STATUS = {
    0: "MOE_OK", 1: "MOE_ERR_INVALID_ARG", 2: "MOE_ERR_CUDA", 3: "MOE_ERR_NOT_SYMMETRIC",
    4: "MOE_ERR_OUT_OF_MEMORY", 5: "MOE_ERR_RECV_OVERFLOW", 6: "MOE_ERR_TIMEOUT",
    7: "MOE_ERR_NOT_READY",
}


class MoEError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {_STATUS.get(code, code)}")
        self.code = code


class moe_shape(ctypes.Structure):
    _fields_ = [
        ("T_local", ctypes.c_int64),
        ("d", ctypes.c_int32),
        ("E", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("f", ctypes.c_int32),
        ("E_shared", ctypes.c_int32),
        ("capacity_factor", ctypes.c_float),
        ("ep_size", ctypes.c_int32),
        ("ep_rank", ctypes.c_int32),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python paper_2605_05049_b200/build.py` "
            "(there is no CPU or eager fallback)")
    return ctypes.CDLL(LIB_PATH)


_lib = _load()
P = ctypes.c_void_p
I32, I64 = ctypes.c_int32, ctypes.c_int64

_SIGS = {
    "moe_ctx_create": [ctypes.POINTER(P), ctypes.POINTER(moe_shape), ctypes.c_int, ctypes.c_size_t],
    "moe_ctx_export_handle": [P, P],
    "moe_ctx_open_peers": [P, P],
    "moe_symm_alloc": [P, ctypes.c_size_t, ctypes.POINTER(P)],
    "moe_symm_free": [P, P],
    "moe_symm_fingerprint": [P, P],
    "moe_ctx_device_bytes": [P, P, P, P],
    "moe_ctx_verify_symmetric": [P, P],
    "moe_migrate": [P, P, P, P, P, ctypes.c_size_t, P],
    "moe_all_to_all": [P, P, P, ctypes.c_size_t, P],
    "moe_ctx_get_device_error": [P],
    "moe_ctx_set_sm_limits": [P, ctypes.c_int, ctypes.c_int],
    "moe_ctx_set_placement": [P, P],
    "moe_rebalance": [P, I32, I32, I32, P, P],
    "moe_load_imbalance": [P, P, I32, I32, P],
    "moe_ctx_destroy": [P],
    "moe_router_logits": [P, P, P, P, P, P],
    "moe_router_logits_bwd": [P, P, P, P, P, P, ctypes.c_int, P],
    "moe_route": [P, P, P, P, P],
    "moe_route_bwd": [P, P, P, P, P, P, P],
    "moe_permute": [P, P, P, P, P, P, P],
    "moe_permute_dispatch_local": [P, P, P, P, P, P, P, P],
    "moe_unpermute": [P, P, P, P, P, P, P],
    "moe_combine_bwd_local": [P, P, P, P, P, P, P, P, P],
    "moe_permute_bwd": [P, P, P, P, P, P, P],
    "moe_permute_bwd_router": [P, P, P, P, P, P, P, P, P],
    "moe_dispatch": [P, P, P, P, P, P],
    "moe_dispatch_bwd": [P, P, P, P, P],
    "moe_expert_ffn": [P, P, P, I32, I64, I32, P, P, P, P, P],
    "moe_expert_ffn_bwd": [P, P, P, I32, I64, I32, P, P, P, P, P, P, P, P, ctypes.c_int, P],
    "moe_expert_ffn_combine": [P, P, P, P, P, P, P, P, P, P, P, P],
    "moe_expert_ffn_bwd_dispatch": [P, P, P, P, P, P, P, P, P, P, P, ctypes.c_int, P],
    "moe_combine": [P, P, P, P, P, P, P, P, P],
    "moe_combine_bwd": [P, P, P, P, P, P, P, P, P],
    "moe_dispatch_range": [P, P, P, P, P, I32, I32, P],
    "moe_combine_bwd_range": [P, P, P, P, P, P, P, P, I32, I32, P],
    "moe_expert_ffn_up": [P, P, P, I32, I32, P, P, P],
    "moe_dispatch_expert_ffn_up": [P, P, P, P, P, P, P, P],
    "moe_combine_bwd_expert_ffn_dh": [P] * 12,
    "moe_expert_ffn_down_combine": [P, P, P, P, P, P, P, P, P, P],
    "moe_expert_ffn_bwd_dh": [P, P, I32, I32, P, P, P, P, P],
    "moe_expert_ffn_bwd_dx_dispatch": [P, P, P, P, P, P, P, P, P, P, ctypes.c_int, P],
    "moe_dedup_pairs": [P, P, P, P, P, P],
    "moe_dedup_dispatch": [P] + [P] * 14,
    "moe_dedup_combine": [P] * 10,
    "moe_dedup_combine_bwd": [P] * 12,
    "moe_dedup_dispatch_bwd": [P] * 12,
    "moe_dedup_combine_bwd_ys": [P] * 14,
    "moe_pipeline_1f1b": [I32, I32, I32, P, I32, P],
    "moe_dedup_permute_bwd_router": [P] * 9,
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
for _name in ("moe_capacity", "moe_recv_rows_max", "moe_layout_ints", "moe_dedup_pair_rows_max",
              "moe_dedup_token_rows_max"):
    getattr(_lib, _name).argtypes = [ctypes.POINTER(moe_shape)]
    getattr(_lib, _name).restype = I64
_lib.moe_layout_offset.argtypes = [ctypes.POINTER(moe_shape), ctypes.c_int]
_lib.moe_layout_offset.restype = I64
_lib.moe_status_string.argtypes = [ctypes.c_int]
_lib.moe_status_string.restype = ctypes.c_char_p

EXPORTED = sorted(list(_SIGS) + ["moe_capacity", "moe_recv_rows_max", "moe_layout_ints",
                                 "moe_layout_offset", "moe_status_string",
                                 "moe_dedup_pair_rows_max", "moe_dedup_token_rows_max"])


def _check(fn, code):
    if code != 0:
        raise MoEError(fn, code)


def _ptr(t, dtype=None, name="tensor"):
    """Device pointer of a contiguous tensor (None -> NULL)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor (libmoe has no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return t.data_ptr()


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def make_shape(T_local, d, E, k, f, E_shared=0, capacity_factor=1.25, ep_size=1, ep_rank=0):
    return moe_shape(int(T_local), int(d), int(E), int(k), int(f), int(E_shared),
                     float(capacity_factor), int(ep_size), int(ep_rank))


def moe_capacity(shape):
    return _lib.moe_capacity(ctypes.byref(shape))


def moe_recv_rows_max(shape):
    return _lib.moe_recv_rows_max(ctypes.byref(shape))


def moe_layout_ints(shape):
    return _lib.moe_layout_ints(ctypes.byref(shape))


def moe_dedup_pair_rows_max(shape):
    return _lib.moe_dedup_pair_rows_max(ctypes.byref(shape))


def moe_dedup_token_rows_max(shape):
    return _lib.moe_dedup_token_rows_max(ctypes.byref(shape))


def moe_layout_offset(shape, field):
    return _lib.moe_layout_offset(ctypes.byref(shape), int(field))


def moe_rebalance(loads, ep, placement=None, max_iters=100):
    """Alg. 2 in libmoe: returns (new placement list, swap count)."""
    E = len(loads)
    ld = (ctypes.c_int64 * E)(*[int(v) for v in loads])
    pl = (ctypes.c_int32 * E)(*([int(v) for v in placement] if placement is not None else range(E)))
    n = ctypes.c_int32(0)
    _check("moe_rebalance", _lib.moe_rebalance(ld, E, int(ep), int(max_iters), pl, ctypes.byref(n)))
    return list(pl), n.value


def moe_migrate(ctx, old_placement, new_placement, src, dst, stream=None):
    """src, dst: symmetric tensors [E_l, ...] (same shape and dtype); one expert per row."""
    if src.shape != dst.shape or src.dtype != dst.dtype:
        raise ValueError("moe_migrate: src and dst must have the same shape and dtype")
    E = len(old_placement)
    o = (ctypes.c_int32 * E)(*[int(v) for v in old_placement])
    n = (ctypes.c_int32 * E)(*[int(v) for v in new_placement])
    per = src[0].numel() * src.element_size() if src.shape[0] else 0
    _check("moe_migrate", _lib.moe_migrate(ctx.handle, o, n, _ptr(src, name="src"),
                                           _ptr(dst, name="dst"), per, _stream(stream)))


def moe_all_to_all(ctx, send, recv, stream=None):
    """send [EP, n] (local), recv [EP, n] symmetric, same dtype: recv chunk r on rank q = send
    chunk q on rank r."""
    per = send[0].numel() * send.element_size() if send.shape[0] else 0
    _check("moe_all_to_all", _lib.moe_all_to_all(ctx.handle, _ptr(send, name="send"),
                                                 _ptr(recv, name="recv"), per, _stream(stream)))


def moe_load_imbalance(loads, placement, ep):
    """max / mean of the EP ranks' routed rows under a placement (migration trigger)."""
    E = len(loads)
    ld = (ctypes.c_int64 * E)(*[int(v) for v in loads])
    pl = (ctypes.c_int32 * E)(*[int(v) for v in placement])
    out = ctypes.c_double(0.0)
    _check("moe_load_imbalance", _lib.moe_load_imbalance(ld, pl, E, int(ep), ctypes.byref(out)))
    return out.value


def moe_status_string(code):
    return _lib.moe_status_string(int(code)).decode()


class _CudaArray:
    """Exposes a raw device pointer through __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class Context:
    """Owns a moe_ctx (symmetric heap, peer table, flags).  One per (process, GPU)."""

    def __init__(self, shape: moe_shape, device: int, heap_bytes: int):
        self.shape = shape
        self.device = int(device)
        self._h = P()
        _check("moe_ctx_create", _lib.moe_ctx_create(ctypes.byref(self._h), ctypes.byref(shape),
                                                     self.device, int(heap_bytes)))
        self._views = []

    @property
    def handle(self):
        return self._h

    def export_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(MOE_IPC_HANDLE_BYTES)
        _check("moe_ctx_export_handle", _lib.moe_ctx_export_handle(self._h, buf))
        return buf.raw

    def open_peers(self, handles: bytes):
        buf = ctypes.create_string_buffer(bytes(handles), len(handles))
        _check("moe_ctx_open_peers", _lib.moe_ctx_open_peers(self._h, buf))

    def symm_empty(self, shape, dtype) -> torch.Tensor:
        """A tensor in the symmetric heap (collective: same calls on every rank)."""
        numel = 1
        for s in shape:
            numel *= int(s)
        elem = torch.empty((), dtype=dtype).element_size()
        nbytes = max(numel * elem, 1)
        p = P()
        _check("moe_symm_alloc", _lib.moe_symm_alloc(self._h, nbytes, ctypes.byref(p)))
        raw = torch.as_tensor(_CudaArray(p.value, nbytes), device=f"cuda:{self.device}")
        t = raw[: numel * elem].view(dtype).view(*shape)
        self._views.append(raw)
        return t

    def symm_free(self, t: torch.Tensor):
        """Releases the LAST symmetric allocation (LIFO; collective)."""
        _check("moe_symm_free", _lib.moe_symm_free(self._h, P(t.data_ptr())))
        self._views.pop()

    def device_bytes(self):
        """(heap bytes, heap bytes allocated, total device bytes of the ctx)."""
        h, u, t = ctypes.c_size_t(0), ctypes.c_size_t(0), ctypes.c_size_t(0)
        _check("moe_ctx_device_bytes", _lib.moe_ctx_device_bytes(
            self._h, ctypes.byref(h), ctypes.byref(u), ctypes.byref(t)))
        return h.value, u.value, t.value

    def fingerprint(self) -> bytes:
        out = ctypes.c_uint64(0)
        _check("moe_symm_fingerprint", _lib.moe_symm_fingerprint(self._h, ctypes.byref(out)))
        return int(out.value).to_bytes(8, "little")

    def verify_symmetric(self, fingerprints: bytes):
        """fingerprints: the all-gathered 8-byte fingerprints in rank order."""
        n = len(fingerprints) // 8
        arr = (ctypes.c_uint64 * n)(*[int.from_bytes(fingerprints[8 * i:8 * i + 8], "little")
                                      for i in range(n)])
        _check("moe_ctx_verify_symmetric", _lib.moe_ctx_verify_symmetric(self._h, arr))

    def set_placement(self, placement):
        """placement: sequence of E ints (expert -> global slot), collective."""
        arr = (ctypes.c_int32 * len(placement))(*[int(v) for v in placement])
        _check("moe_ctx_set_placement", _lib.moe_ctx_set_placement(self._h, arr))

    def set_sm_limits(self, gemm_sms: int, comm_sms: int):
        _check("moe_ctx_set_sm_limits", _lib.moe_ctx_set_sm_limits(self._h, int(gemm_sms),
                                                                   int(comm_sms)))

    def device_error(self):
        return _lib.moe_ctx_get_device_error(self._h)

    def check_device_error(self):
        _check("moe_ctx_get_device_error", self.device_error())

    def close(self):
        if self._h:
            self._views.clear()
            _lib.moe_ctx_destroy(self._h)
            self._h = P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


BF16, F32, I32T = torch.bfloat16, torch.float32, torch.int32


def moe_router_logits(ctx, x, w_r, bias, logits, stream=None):
    _check("moe_router_logits", _lib.moe_router_logits(
        ctx.handle, _ptr(x, BF16, "x"), _ptr(w_r, BF16, "w_r"), _ptr(bias, F32, "bias"),
        _ptr(logits, F32, "logits"), _stream(stream)))


def moe_router_logits_bwd(ctx, x, w_r, dlogits, dx_router, dw_r, accumulate=False, stream=None):
    _check("moe_router_logits_bwd", _lib.moe_router_logits_bwd(
        ctx.handle, _ptr(x, BF16, "x"), _ptr(w_r, BF16, "w_r"), _ptr(dlogits, F32, "dlogits"),
        _ptr(dx_router, F32, "dx_router"), _ptr(dw_r, F32, "dw_r"), int(bool(accumulate)),
        _stream(stream)))


def moe_route(ctx, logits, topk_idx, gates, stream=None):
    _check("moe_route", _lib.moe_route(ctx.handle, _ptr(logits, F32, "logits"),
                                       _ptr(topk_idx, I32T, "topk_idx"), _ptr(gates, F32, "gates"),
                                       _stream(stream)))


def moe_route_bwd(ctx, logits, topk_idx, gates, dgates, dlogits, stream=None):
    _check("moe_route_bwd", _lib.moe_route_bwd(
        ctx.handle, _ptr(logits, F32, "logits"), _ptr(topk_idx, I32T, "topk_idx"),
        _ptr(gates, F32, "gates"), _ptr(dgates, F32, "dgates"), _ptr(dlogits, F32, "dlogits"),
        _stream(stream)))


def moe_permute(ctx, x, topk_idx, counts, dest_row, xs, stream=None):
    _check("moe_permute", _lib.moe_permute(
        ctx.handle, _ptr(x, BF16, "x"), _ptr(topk_idx, I32T, "topk_idx"), _ptr(counts, I32T, "counts"),
        _ptr(dest_row, I32T, "dest_row"), _ptr(xs, BF16, "xs"), _stream(stream)))


def moe_permute_dispatch_local(ctx, x, topk_idx, counts, dest_row, layout, xr, stream=None):
    _check("moe_permute_dispatch_local", _lib.moe_permute_dispatch_local(
        ctx.handle, _ptr(x, BF16, "x"), _ptr(topk_idx, I32T, "topk_idx"),
        _ptr(counts, I32T, "counts"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(layout, I32T, "layout"), _ptr(xr, BF16, "xr"), _stream(stream)))


def moe_unpermute(ctx, rows, gates, dest_row, y_extra, y, stream=None):
    _check("moe_unpermute", _lib.moe_unpermute(
        ctx.handle, _ptr(rows, BF16, "rows"), _ptr(gates, F32, "gates"),
        _ptr(dest_row, I32T, "dest_row"), _ptr(y_extra, BF16, "y_extra"), _ptr(y, BF16, "y"),
        _stream(stream)))


def moe_combine_bwd_local(ctx, dy, gates, dest_row, out, layout, dgates, dout_r, stream=None):
    _check("moe_combine_bwd_local", _lib.moe_combine_bwd_local(
        ctx.handle, _ptr(dy, BF16, "dy"), _ptr(gates, F32, "gates"),
        _ptr(dest_row, I32T, "dest_row"), _ptr(out, BF16, "out"), _ptr(layout, I32T, "layout"),
        _ptr(dgates, F32, "dgates"), _ptr(dout_r, BF16, "dout_r"), _stream(stream)))


def moe_permute_bwd(ctx, dxs, dest_row, dx_acc, dx_extra, dx, stream=None):
    _check("moe_permute_bwd", _lib.moe_permute_bwd(
        ctx.handle, _ptr(dxs, BF16, "dxs"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(dx_acc, F32, "dx_acc"), _ptr(dx_extra, BF16, "dx_extra"), _ptr(dx, BF16, "dx"),
        _stream(stream)))


def moe_permute_bwd_router(ctx, dxs, dest_row, topk_idx, dlogits, w_r, dx_extra, dx, stream=None):
    _check("moe_permute_bwd_router", _lib.moe_permute_bwd_router(
        ctx.handle, _ptr(dxs, BF16, "dxs"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(topk_idx, I32T, "topk_idx"), _ptr(dlogits, F32, "dlogits"), _ptr(w_r, BF16, "w_r"),
        _ptr(dx_extra, BF16, "dx_extra"), _ptr(dx, BF16, "dx"), _stream(stream)))


def moe_dispatch(ctx, xs, counts, layout, xr, stream=None):
    _check("moe_dispatch", _lib.moe_dispatch(
        ctx.handle, _ptr(xs, BF16, "xs"), _ptr(counts, I32T, "counts"), _ptr(layout, I32T, "layout"),
        _ptr(xr, BF16, "xr"), _stream(stream)))


def moe_dispatch_bwd(ctx, dxr, layout, dxs, stream=None):
    _check("moe_dispatch_bwd", _lib.moe_dispatch_bwd(
        ctx.handle, _ptr(dxr, BF16, "dxr"), _ptr(layout, I32T, "layout"), _ptr(dxs, BF16, "dxs"),
        _stream(stream)))


def moe_expert_ffn(ctx, xr, group_rows, n_groups, rows_cap, f, w_gu, w_down, g_u_h, out, stream=None):
    _check("moe_expert_ffn", _lib.moe_expert_ffn(
        ctx.handle, _ptr(xr, BF16, "xr"), _ptr(group_rows, I32T, "group_rows"), int(n_groups),
        int(rows_cap), int(f), _ptr(w_gu, BF16, "w_gu"), _ptr(w_down, BF16, "w_down"),
        _ptr(g_u_h, BF16, "g_u_h"), _ptr(out, BF16, "out"), _stream(stream)))


def moe_expert_ffn_bwd(ctx, xr, group_rows, n_groups, rows_cap, f, w_gu, w_down, g_u_h, dout, dgu,
                       dxr, dw_gu, dw_down, accumulate=False, stream=None):
    _check("moe_expert_ffn_bwd", _lib.moe_expert_ffn_bwd(
        ctx.handle, _ptr(xr, BF16, "xr"), _ptr(group_rows, I32T, "group_rows"), int(n_groups),
        int(rows_cap), int(f), _ptr(w_gu, BF16, "w_gu"), _ptr(w_down, BF16, "w_down"),
        _ptr(g_u_h, BF16, "g_u_h"), _ptr(dout, BF16, "dout"), _ptr(dgu, BF16, "dgu"),
        _ptr(dxr, BF16, "dxr"), _ptr(dw_gu, F32, "dw_gu"), _ptr(dw_down, F32, "dw_down"),
        int(bool(accumulate)), _stream(stream)))


def moe_expert_ffn_combine(ctx, xr, layout, w_gu, w_down, g_u_h, ys, gates, dest_row, y_extra, y,
                           stream=None):
    _check("moe_expert_ffn_combine", _lib.moe_expert_ffn_combine(
        ctx.handle, _ptr(xr, BF16, "xr"), _ptr(layout, I32T, "layout"), _ptr(w_gu, BF16, "w_gu"),
        _ptr(w_down, BF16, "w_down"), _ptr(g_u_h, BF16, "g_u_h"), _ptr(ys, BF16, "ys"),
        _ptr(gates, F32, "gates"), _ptr(dest_row, I32T, "dest_row"), _ptr(y_extra, BF16, "y_extra"),
        _ptr(y, BF16, "y"), _stream(stream)))


def moe_expert_ffn_bwd_dispatch(ctx, xr, layout, w_gu, w_down, g_u_h, dout, dgu, dxs, dw_gu, dw_down,
                                accumulate=False, stream=None):
    _check("moe_expert_ffn_bwd_dispatch", _lib.moe_expert_ffn_bwd_dispatch(
        ctx.handle, _ptr(xr, BF16, "xr"), _ptr(layout, I32T, "layout"), _ptr(w_gu, BF16, "w_gu"),
        _ptr(w_down, BF16, "w_down"), _ptr(g_u_h, BF16, "g_u_h"), _ptr(dout, BF16, "dout"),
        _ptr(dgu, BF16, "dgu"), _ptr(dxs, BF16, "dxs"), _ptr(dw_gu, F32, "dw_gu"),
        _ptr(dw_down, F32, "dw_down"), int(bool(accumulate)), _stream(stream)))


def moe_combine(ctx, out, layout, ys, gates, dest_row, y_extra, y, stream=None):
    _check("moe_combine", _lib.moe_combine(
        ctx.handle, _ptr(out, BF16, "out"), _ptr(layout, I32T, "layout"), _ptr(ys, BF16, "ys"),
        _ptr(gates, F32, "gates"), _ptr(dest_row, I32T, "dest_row"), _ptr(y_extra, BF16, "y_extra"),
        _ptr(y, BF16, "y"), _stream(stream)))


def moe_combine_bwd(ctx, dy, gates, dest_row, ys, layout, dgates, dout_r, stream=None):
    _check("moe_combine_bwd", _lib.moe_combine_bwd(
        ctx.handle, _ptr(dy, BF16, "dy"), _ptr(gates, F32, "gates"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(ys, BF16, "ys"), _ptr(layout, I32T, "layout"), _ptr(dgates, F32, "dgates"),
        _ptr(dout_r, BF16, "dout_r"), _stream(stream)))


# ---- NEXT-1 chunked overlap: slot-range transfers and the expert GEMM phases (include/moe.h)
def moe_dispatch_range(ctx, xs, counts, layout, xr, slot_begin, slot_end, stream=None):
    _check("moe_dispatch_range", _lib.moe_dispatch_range(
        ctx.handle, _ptr(xs, BF16, "xs"), _ptr(counts, I32T, "counts"), _ptr(layout, I32T, "layout"),
        _ptr(xr, BF16, "xr"), int(slot_begin), int(slot_end), _stream(stream)))


def moe_combine_bwd_range(ctx, dy, gates, dest_row, ys, layout, dgates, dout_r, slot_begin,
                          slot_end, stream=None):
    _check("moe_combine_bwd_range", _lib.moe_combine_bwd_range(
        ctx.handle, _ptr(dy, BF16, "dy"), _ptr(gates, F32, "gates"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(ys, BF16, "ys"), _ptr(layout, I32T, "layout"), _ptr(dgates, F32, "dgates"),
        _ptr(dout_r, BF16, "dout_r"), int(slot_begin), int(slot_end), _stream(stream)))


def moe_expert_ffn_up(ctx, xr, layout, slot_begin, slot_end, w_gu, g_u_h, stream=None):
    _check("moe_expert_ffn_up", _lib.moe_expert_ffn_up(
        ctx.handle, _ptr(xr, BF16, "xr"), _ptr(layout, I32T, "layout"), int(slot_begin),
        int(slot_end), _ptr(w_gu, BF16, "w_gu"), _ptr(g_u_h, BF16, "g_u_h"), _stream(stream)))


def moe_dispatch_expert_ffn_up(ctx, xs, counts, layout, xr, w_gu, g_u_h, stream=None):
    _check("moe_dispatch_expert_ffn_up", _lib.moe_dispatch_expert_ffn_up(
        ctx.handle, _ptr(xs, BF16, "xs"), _ptr(counts, I32T, "counts"),
        _ptr(layout, I32T, "layout"), _ptr(xr, BF16, "xr"), _ptr(w_gu, BF16, "w_gu"),
        _ptr(g_u_h, BF16, "g_u_h"), _stream(stream)))


def moe_combine_bwd_expert_ffn_dh(ctx, dy, gates, dest_row, ys, layout, dgates, dout_r, w_down,
                                  g_u_h, dgu, stream=None):
    _check("moe_combine_bwd_expert_ffn_dh", _lib.moe_combine_bwd_expert_ffn_dh(
        ctx.handle, _ptr(dy, BF16, "dy"), _ptr(gates, F32, "gates"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(ys, BF16, "ys"), _ptr(layout, I32T, "layout"), _ptr(dgates, F32, "dgates"),
        _ptr(dout_r, BF16, "dout_r"), _ptr(w_down, BF16, "w_down"), _ptr(g_u_h, BF16, "g_u_h"),
        _ptr(dgu, BF16, "dgu"), _stream(stream)))


def moe_expert_ffn_down_combine(ctx, layout, w_down, g_u_h, ys, gates, dest_row, y_extra, y,
                                stream=None):
    _check("moe_expert_ffn_down_combine", _lib.moe_expert_ffn_down_combine(
        ctx.handle, _ptr(layout, I32T, "layout"), _ptr(w_down, BF16, "w_down"),
        _ptr(g_u_h, BF16, "g_u_h"), _ptr(ys, BF16, "ys"), _ptr(gates, F32, "gates"),
        _ptr(dest_row, I32T, "dest_row"), _ptr(y_extra, BF16, "y_extra"), _ptr(y, BF16, "y"),
        _stream(stream)))


def moe_expert_ffn_bwd_dh(ctx, layout, slot_begin, slot_end, w_down, g_u_h, dout, dgu, stream=None):
    _check("moe_expert_ffn_bwd_dh", _lib.moe_expert_ffn_bwd_dh(
        ctx.handle, _ptr(layout, I32T, "layout"), int(slot_begin), int(slot_end),
        _ptr(w_down, BF16, "w_down"), _ptr(g_u_h, BF16, "g_u_h"), _ptr(dout, BF16, "dout"),
        _ptr(dgu, BF16, "dgu"), _stream(stream)))


def moe_expert_ffn_bwd_dx_dispatch(ctx, xr, layout, w_gu, g_u_h, dout, dgu, dxs, dw_gu, dw_down,
                                   accumulate=False, stream=None):
    _check("moe_expert_ffn_bwd_dx_dispatch", _lib.moe_expert_ffn_bwd_dx_dispatch(
        ctx.handle, _ptr(xr, BF16, "xr"), _ptr(layout, I32T, "layout"), _ptr(w_gu, BF16, "w_gu"),
        _ptr(g_u_h, BF16, "g_u_h"), _ptr(dout, BF16, "dout"), _ptr(dgu, BF16, "dgu"),
        _ptr(dxs, BF16, "dxs"), _ptr(dw_gu, F32, "dw_gu"), _ptr(dw_down, F32, "dw_down"),
        int(bool(accumulate)), _stream(stream)))


# ---- NEXT-4 deduplicated all-to-all (include/moe.h, reading R18)
def moe_dedup_pairs(ctx, topk_idx, dest_row, pdest, ntok, stream=None):
    _check("moe_dedup_pairs", _lib.moe_dedup_pairs(
        ctx.handle, _ptr(topk_idx, I32T, "topk_idx"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(pdest, I32T, "pdest"), _ptr(ntok, I32T, "ntok"), _stream(stream)))


def moe_dedup_dispatch(ctx, x, counts, ntok, pdest, dest_row, topk_idx, gates, layout, dlayout,
                       xt, rlist, glist, xr, stream=None):
    _check("moe_dedup_dispatch", _lib.moe_dedup_dispatch(
        ctx.handle, _ptr(x, BF16, "x"), _ptr(counts, I32T, "counts"), _ptr(ntok, I32T, "ntok"),
        _ptr(pdest, I32T, "pdest"), _ptr(dest_row, I32T, "dest_row"),
        _ptr(topk_idx, I32T, "topk_idx"), _ptr(gates, F32, "gates"), _ptr(layout, I32T, "layout"),
        _ptr(dlayout, I32T, "dlayout"), _ptr(xt, BF16, "xt"), _ptr(rlist, I32T, "rlist"),
        _ptr(glist, F32, "glist"), _ptr(xr, BF16, "xr"), _stream(stream)))


def moe_dedup_combine(ctx, out, dlayout, rlist, glist, pdest, y_extra, part, y, stream=None):
    _check("moe_dedup_combine", _lib.moe_dedup_combine(
        ctx.handle, _ptr(out, BF16, "out"), _ptr(dlayout, I32T, "dlayout"),
        _ptr(rlist, I32T, "rlist"), _ptr(glist, F32, "glist"), _ptr(pdest, I32T, "pdest"),
        _ptr(y_extra, BF16, "y_extra"), _ptr(part, BF16, "part"), _ptr(y, BF16, "y"),
        _stream(stream)))


def moe_dedup_combine_bwd(ctx, dy, pdest, layout, dlayout, rlist, glist, out, dyt, dg_own, dout_r,
                          stream=None):
    _check("moe_dedup_combine_bwd", _lib.moe_dedup_combine_bwd(
        ctx.handle, _ptr(dy, BF16, "dy"), _ptr(pdest, I32T, "pdest"), _ptr(layout, I32T, "layout"),
        _ptr(dlayout, I32T, "dlayout"), _ptr(rlist, I32T, "rlist"), _ptr(glist, F32, "glist"),
        _ptr(out, BF16, "out"), _ptr(dyt, BF16, "dyt"), _ptr(dg_own, F32, "dg_own"),
        _ptr(dout_r, BF16, "dout_r"), _stream(stream)))


def moe_dedup_dispatch_bwd(ctx, dxr, dlayout, rlist, dg_own, pdest, dest_row, topk_idx, dxpart,
                           dgpart, dgates, stream=None):
    _check("moe_dedup_dispatch_bwd", _lib.moe_dedup_dispatch_bwd(
        ctx.handle, _ptr(dxr, BF16, "dxr"), _ptr(dlayout, I32T, "dlayout"),
        _ptr(rlist, I32T, "rlist"), _ptr(dg_own, F32, "dg_own"), _ptr(pdest, I32T, "pdest"),
        _ptr(dest_row, I32T, "dest_row"), _ptr(topk_idx, I32T, "topk_idx"),
        _ptr(dxpart, BF16, "dxpart"), _ptr(dgpart, F32, "dgpart"), _ptr(dgates, F32, "dgates"),
        _stream(stream)))


def moe_dedup_permute_bwd_router(ctx, dxpart, pdest, topk_idx, dlogits, w_r, dx_extra, dx,
                                 stream=None):
    _check("moe_dedup_permute_bwd_router", _lib.moe_dedup_permute_bwd_router(
        ctx.handle, _ptr(dxpart, BF16, "dxpart"), _ptr(pdest, I32T, "pdest"),
        _ptr(topk_idx, I32T, "topk_idx"), _ptr(dlogits, F32, "dlogits"), _ptr(w_r, BF16, "w_r"),
        _ptr(dx_extra, BF16, "dx_extra"), _ptr(dx, BF16, "dx"), _stream(stream)))


def moe_dedup_combine_bwd_ys(ctx, dy, gates, dest_row, ys, pdest, layout, dlayout, rlist, glist,
                             dyt, dgates, dout_r, stream=None):
    _check("moe_dedup_combine_bwd_ys", _lib.moe_dedup_combine_bwd_ys(
        ctx.handle, _ptr(dy, BF16, "dy"), _ptr(gates, F32, "gates"),
        _ptr(dest_row, I32T, "dest_row"), _ptr(ys, BF16, "ys"), _ptr(pdest, I32T, "pdest"),
        _ptr(layout, I32T, "layout"), _ptr(dlayout, I32T, "dlayout"), _ptr(rlist, I32T, "rlist"),
        _ptr(glist, F32, "glist"), _ptr(dyt, BF16, "dyt"), _ptr(dgates, F32, "dgates"),
        _ptr(dout_r, BF16, "dout_r"), _stream(stream)))


# ---- NEXT-3 PP x EP executor: the 1F1B op list of one stage (host code in libmoe)
PIPE_FORWARD, PIPE_BACKWARD = 0, 1


def moe_pipeline_1f1b(pp, stage, n_micro):
    """[(PIPE_FORWARD | PIPE_BACKWARD, micro-batch), ...] of `stage` (reading R19)."""
    cap = max(2 * int(n_micro), 1)
    ops = (ctypes.c_int32 * (2 * cap))()
    n = ctypes.c_int32(0)
    _check("moe_pipeline_1f1b", _lib.moe_pipeline_1f1b(int(pp), int(stage), int(n_micro), ops,
                                                       cap, ctypes.byref(n)))
    return [(ops[2 * i], ops[2 * i + 1]) for i in range(n.value)]

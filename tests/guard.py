"""Guard bands around every device buffer of a layer: an out-of-bounds write check that needs
no tooling (compute-sanitizer is closed on the GPU pool).

Inside `guarded()`, every `torch.empty` / `torch.zeros` on a CUDA device returns the middle of a
larger allocation whose GUARD bytes on each side hold a canary byte pattern, and every
symmetric-heap allocation (`Context.symm_empty`) is followed by a canary allocation of GUARD
bytes.  `check()` reports every guard whose bytes changed -- a kernel that writes past the end
(or before the start) of any buffer it was given, or a peer that stores past a symmetric
buffer, flips canary bytes.  Allocation order is unchanged, so the symmetric fingerprints of
the ranks still agree.
"""
from __future__ import annotations

import contextlib

import torch

GUARD = 4096     # bytes on each side
CANARY = 0xA5


class Guards:
    def __init__(self):
        self.regions = []   # (name, uint8 tensor view of a guard band)

    def check(self):
        torch.cuda.synchronize()
        return [name for name, g in self.regions if not bool((g == CANARY).all())]


@contextlib.contextmanager
def guarded():
    from paper_2605_05049_b200 import _lib as L
    gs = Guards()
    orig_empty, orig_zeros = torch.empty, torch.zeros
    orig_symm = L.Context.symm_empty

    def _alloc(shape, dtype, device, fill_zero):
        if isinstance(shape, int):
            shape = (shape,)
        numel = 1
        for s in shape:
            numel *= int(s)
        esize = orig_empty((), dtype=dtype).element_size()
        nbytes = numel * esize
        raw = orig_empty((GUARD + nbytes + GUARD,), dtype=torch.uint8, device=device)
        raw.fill_(CANARY)
        gs.regions.append((f"torch{tuple(shape)}:{dtype}:lo", raw[:GUARD]))
        gs.regions.append((f"torch{tuple(shape)}:{dtype}:hi", raw[GUARD + nbytes:]))
        t = raw[GUARD:GUARD + nbytes].view(dtype).view(*shape)
        if fill_zero:
            t.zero_()
        return t

    def empty(*shape, dtype=None, device=None, **kw):
        if len(shape) == 1 and isinstance(shape[0], (tuple, list, torch.Size)):
            shape = tuple(shape[0])
        dev = torch.device(device) if device is not None else None
        if dev is None or dev.type != "cuda" or kw:
            return orig_empty(tuple(shape), dtype=dtype, device=device, **kw)
        return _alloc(shape, dtype or torch.float32, dev, False)

    def zeros(*shape, dtype=None, device=None, **kw):
        if len(shape) == 1 and isinstance(shape[0], (tuple, list, torch.Size)):
            shape = tuple(shape[0])
        dev = torch.device(device) if device is not None else None
        if dev is None or dev.type != "cuda" or kw:
            return orig_zeros(tuple(shape), dtype=dtype, device=device, **kw)
        return _alloc(shape, dtype or torch.float32, dev, True)

    def symm_empty(self, shape, dtype):
        t = orig_symm(self, shape, dtype)
        g = orig_symm(self, (GUARD,), torch.uint8)
        g.fill_(CANARY)
        gs.regions.append((f"symm{tuple(shape)}:{dtype}:hi", g))
        return t

    torch.empty, torch.zeros = empty, zeros
    L.Context.symm_empty = symm_empty
    try:
        yield gs
    finally:
        torch.empty, torch.zeros = orig_empty, orig_zeros
        L.Context.symm_empty = orig_symm

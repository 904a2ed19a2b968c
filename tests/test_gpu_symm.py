"""Symmetric-heap safety checks of the C ABI: allocation fingerprints, sized
destination checks of the collectives, LIFO free, and T_local = 0 accepted with NULL token
buffers."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ctx(T=64, d=128, E=8, k=2, f=256, heap=1 << 22):
    from paper_2605_05049_b200 import _lib as L
    shape = L.make_shape(T, d, E, k, f, 0, 1.25, 1, 0)
    return L, shape, L.Context(shape, 0, heap)


def test_fingerprint_and_verify():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    L, shape, ctx = _ctx()
    f0 = ctx.fingerprint()
    ctx.symm_empty((128, 128), torch.bfloat16)
    f1 = ctx.fingerprint()
    assert f1 != f0
    ctx.verify_symmetric(f1)                      # one rank, same sequence
    other = (int.from_bytes(f1, "little") ^ 1).to_bytes(8, "little")
    with pytest.raises(L.MoEError) as e:
        ctx.verify_symmetric(other)
    assert e.value.code == 3                      # MOE_ERR_NOT_SYMMETRIC
    ctx.close()


def test_collective_destination_must_fit_one_allocation():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    L, shape, ctx = _ctx()
    R = L.moe_recv_rows_max(shape)
    small = ctx.symm_empty((R // 2, 128), torch.bfloat16)        # undersized receive buffer
    xs = torch.zeros((64 * 2, 128), dtype=torch.bfloat16, device="cuda")
    counts = torch.zeros((8,), dtype=torch.int32, device="cuda")
    layout = torch.zeros((L.moe_layout_ints(shape),), dtype=torch.int32, device="cuda")
    with pytest.raises(L.MoEError) as e:
        L.moe_dispatch(ctx, xs, counts, layout, small)
    assert e.value.code == 3
    plain = torch.zeros((R, 128), dtype=torch.bfloat16, device="cuda")   # not symmetric
    with pytest.raises(L.MoEError) as e:
        L.moe_dispatch(ctx, xs, counts, layout, plain)
    assert e.value.code == 3
    big = ctx.symm_empty((R, 128), torch.bfloat16)
    L.moe_dispatch(ctx, xs, counts, layout, big)             # fits: accepted
    torch.cuda.synchronize()
    ctx.check_device_error()
    ctx.close()


def test_symm_free_is_lifo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    L, shape, ctx = _ctx()
    a = ctx.symm_empty((64,), torch.float32)
    b = ctx.symm_empty((64,), torch.float32)
    with pytest.raises(L.MoEError):
        ctx.symm_free(a)                          # not the last allocation
    ctx.symm_free(b)
    c = ctx.symm_empty((64,), torch.float32)      # reuses b's offset
    assert c.data_ptr() == b.data_ptr()
    ctx.close()

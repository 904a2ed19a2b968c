"""Host-side path selection of MoELayer (no GPU): when the NEXT-1 tile-granular transfers
(moe_dispatch_expert_ffn_up, moe_combine_bwd_expert_ffn_dh) replace the separate transfer
kernels, and the launch count bench.py reports for each path."""
import pytest

from paper_2605_05049_b200.layer import LayerDims, MoELayer


def fake_layer(E=64, ep=4, k=6, E_s=0, f=1408, fused=True, dedup=False):
    layer = MoELayer.__new__(MoELayer)   # host attributes only: no ctx, no device buffers
    layer.dims = LayerDims(T_local=16, d=256, E=E, k=k, f=f, E_shared=E_s, ep_size=ep)
    layer.E_l = E // ep
    layer.fs = E_s * f
    layer.fused = fused
    layer.dedup = dedup
    layer.dedup_mode = "dispatch" if dedup else None
    return layer


@pytest.mark.parametrize("E,ep,E_s,fwd,bwd", [
    (8, 4, 0, False, False),     # Mixtral N=4: E_l = 2, the first wave would wait half the transfer
    (8, 1, 0, True, True),       # E_l = 8 (reached at EP = 1 only with local_fast_path False)
    (64, 4, 2, True, False),     # DS-MoE N=4: shared experts keep the separate combine_bwd
    (256, 4, 0, True, True),     # V3-like N=4
    (64, 8, 0, True, True),      # E_l = 8
    (32, 8, 0, False, False),    # E_l = 4
])
def test_tile_overlap_defaults(E, ep, E_s, fwd, bwd):
    layer = fake_layer(E=E, ep=ep, E_s=E_s)
    layer.tile_overlap = None
    layer.tile_overlap_bwd = None
    assert layer._tile_overlap() is fwd
    assert layer._tile_overlap_bwd() is bwd


def test_tile_overlap_forced_and_excluded():
    layer = fake_layer(E=8, ep=4, E_s=2)
    layer.tile_overlap, layer.tile_overlap_bwd = True, True
    assert layer._tile_overlap() and layer._tile_overlap_bwd()
    layer.tile_overlap_bwd = False
    assert layer._tile_overlap() and not layer._tile_overlap_bwd()
    layer.tile_overlap = False
    layer.tile_overlap_bwd = True
    assert not layer._tile_overlap() and not layer._tile_overlap_bwd()   # bwd follows fwd
    for kw in ({"fused": False}, {"dedup": True}):   # step-by-step calls / dedup transfers
        other = fake_layer(E=256, ep=4, **kw)
        other.tile_overlap, other.tile_overlap_bwd = True, True
        assert not other._tile_overlap() and not other._tile_overlap_bwd()


def test_kernel_launches_count_the_fused_transfers():
    """One launch fewer per fused transfer (dispatch + GEMM1, combine_bwd + dgrad-1)."""
    layer = fake_layer(E=256, ep=4, k=8)
    layer.local_fast_path = True
    counts = {}
    for fwd_on, bwd_on in ((False, False), (True, False), (True, True)):
        layer.tile_overlap, layer.tile_overlap_bwd = fwd_on, bwd_on
        counts[(fwd_on, bwd_on)] = (layer.kernel_launches(True, False),
                                    layer.kernel_launches(False, True))
    assert counts[(True, False)] == (counts[(False, False)][0] - 1, counts[(False, False)][1])
    assert counts[(True, True)] == (counts[(False, False)][0] - 1, counts[(False, False)][1] - 1)

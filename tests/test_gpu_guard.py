"""Out-of-bounds write check of the whole layer (tests/guard.py): every device buffer the layer
allocates -- plain and symmetric -- and the inputs sit between canary guard bands; a forward +
backward (twice: buffer reuse) must leave every guard intact.  Covers the EP = 1 local path,
the permute + dispatch path, the transfers fused into GEMM1 / dgrad-1 (tile-granular), the
step-by-step calls, the dedup all-to-alls, drops, k = 1,
shared experts, Zipf skew and T_local = 0 (compute-sanitizer is not available on the pool)."""
import pytest
import torch

import synth
from tests.guard import GUARD, guarded
from tests.test_gpu_layer import CASES, build_layer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,mode", [
    ("tiny", "local"), ("drops", "local"), ("drops", "dispatch"), ("drops", "stepwise"),
    ("dsmoe_small", "local"), ("dsmoe_small", "dedup_all"), ("v3_small_zipf", "dedup_dispatch"),
    ("switch_k1", "local"), ("empty", "local"), ("drops", "tile"), ("dsmoe_small", "tile"),
    ("v3_small_zipf", "tile"), ("empty", "tile")])
def test_layer_guard_bands(name, mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_05049_b200 import MoELayer
    cfg = (synth.MoEConfig("empty", T=0, d=256, E=8, k=2, f=256, cf=1.25, E_s=1)
           if name == "empty" else CASES[name])
    dedup = {"dedup_all": "all", "dedup_dispatch": "dispatch"}.get(mode, False)
    MoELayer.extra_heap_bytes = 64 * GUARD
    try:
        with guarded() as gs:
            layer = build_layer(cfg, dedup=dedup)
            layer.local_fast_path = mode == "local"
            layer.fused = mode != "stepwise"
            # the transfers inside the GEMM launches (NEXT-1) or the separate transfer kernels
            layer.tile_overlap = layer.tile_overlap_bwd = mode == "tile"
            x = torch.empty((cfg.T, cfg.d), dtype=torch.bfloat16, device="cuda")
            dy = torch.empty((cfg.T, cfg.d), dtype=torch.bfloat16, device="cuda")
        x.copy_(synth.tokens(cfg).cuda())
        dy.copy_(synth.grad_output(cfg).cuda())
        for _ in range(2):
            layer.forward(x)
            layer.backward(dy)
        torch.cuda.synchronize()
        layer.ctx.check_device_error()
        bad = gs.check()
        assert not bad, bad
        assert len(gs.regions) > 20
        layer.close()
    finally:
        MoELayer.extra_heap_bytes = 0

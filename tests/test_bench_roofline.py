"""The serial layer roofline bench.py reports against its closed form on
the balanced fixture (every (source, expert) pair carries T_r k / E rows), plain and dedup:
router 3 x 2 T_r d E / pi, GEMMs 18 n d f / pi, HBM passes / beta_hbm, 4 all-to-alls at
max(egress, ingress) / beta_nvl (CPU only: bench's arithmetic, no GPU)."""
import types

import pytest
import torch

import bench


def fake_layer(EP, E, T_r, k, dedup=None, ntok=None):
    E_l = E // EP
    cm = torch.full((EP, E), T_r * k // E, dtype=torch.int32)
    lay = types.SimpleNamespace(
        dims=types.SimpleNamespace(ep_size=EP, T_local=T_r), E_l=E_l,
        layout=cm.reshape(-1), placement=list(range(E)), dedup=dedup is not None,
        dedup_mode=dedup)
    if ntok is not None:
        lay.dlayout = torch.tensor(ntok, dtype=torch.int32).reshape(-1)
    return lay


PEAKS = {"bf16": 1000.0, "bf16_sustained": 800.0, "hbm": 5000.0}


@pytest.mark.parametrize("EP", [1, 2, 4, 8])
def test_plain_layer_roofline_closed_form(EP):
    E, d, f, k, T = 8, 4096, 14336, 2, 8192
    T_r = T // EP
    cfg = types.SimpleNamespace(E=E, d=d, f=f, k=k, E_s=0)
    out = bench.layer_roofline(fake_layer(EP, E, T_r, k), cfg, PEAKS, nvl_gbs=900.0)
    pi, bh, bn, row = 1000e12, 5000e9, 900e9, 2 * d
    recv = send = T_r * k                                 # balanced: every rank the same
    off = T_r * k * (EP - 1) // EP * row                   # egress = ingress
    want = (6 * T_r * d * E / pi + 4 * (T_r * row + send * row) / bh + 4 * off / bn
            + 18 * recv * d * f / pi) * 1e3
    assert out["serial_ms"] == pytest.approx(want, rel=1e-12)
    assert len(out["per_rank_ms"]) == EP


def test_dedup_roofline_uses_pair_rows_on_nvlink():
    """Mode 'dispatch' at EP=4 with one pair per token and owner (k=2 slots on the same owner):
    the dispatch-direction all-to-alls move half the rows of the reverse ones."""
    EP, E, d, f, k, T_r = 4, 16, 2048, 1408, 2, 1024
    cfg = types.SimpleNamespace(E=E, d=d, f=f, k=k, E_s=0)
    ntok = [[T_r // EP] * EP for _ in range(EP)]          # T_r pairs per source, even split
    plain = bench.layer_roofline(fake_layer(EP, E, T_r, k), cfg, PEAKS)
    ded = bench.layer_roofline(fake_layer(EP, E, T_r, k, "dispatch", ntok), cfg, PEAKS)
    row, bn, bh = 2 * d, 900e9, 5000e9
    slots_off = T_r * k * (EP - 1) // EP * row
    pairs_off = T_r * (EP - 1) // EP * row
    recv = send = T_r * k
    # NVLink: two directions drop from slots to pairs; HBM: the permute scatter and the
    # combine_bwd dO writes are replaced by the two expands and the source-side dgates dots
    d_nvl = 2 * (pairs_off - slots_off) / bn
    d_hbm = (2 * (T_r * row + recv * row) + (T_r * row + send * row)
             - 2 * (T_r * row + send * row)) / bh
    assert ded["serial_ms"] - plain["serial_ms"] == pytest.approx((d_nvl + d_hbm) * 1e3, rel=1e-9)


def test_sustained_variant_uses_the_sustained_peak():
    E, d, f, k, T_r = 8, 4096, 14336, 2, 8192
    cfg = types.SimpleNamespace(E=E, d=d, f=f, k=k, E_s=0)
    lay = fake_layer(1, E, T_r, k)
    burst = bench.layer_roofline(lay, cfg, PEAKS)
    sus = bench.layer_roofline(lay, cfg, PEAKS, sustained=True)
    gemm = (6 * T_r * d * E + 18 * T_r * k * d * f)
    hbm = 4 * (T_r * 2 * d + T_r * k * 2 * d) / 5000e9
    assert burst["serial_ms"] == pytest.approx((gemm / 1000e12 + hbm) * 1e3, rel=1e-12)
    assert sus["serial_ms"] == pytest.approx((gemm / 800e12 + hbm) * 1e3, rel=1e-12)

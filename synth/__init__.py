"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no routing, no permutation, no
FFN): it only draws tensors from fixed seeds with the shapes and value
distributions of the paper's workloads (DESIGN.md
"Input recipe").  Both the CUDA path and the fp64 oracle consume the tensors it
returns; neither side generates its own inputs.

Configs (BASELINE.json ``configs``; Table I for the shapes):

* ``tiny``     T=256   d=64   E=8   k=2 f=128   cf=1.25
* ``mixtral``  T=8192  d=4096 E=8   k=2 f=14336 cf=1.25
* ``dsmoe``    T=16384 d=2048 E=64  k=6 f=1408  cf=1.25, 2 shared experts
* ``dsv3``     T=32768 d=7168 E=256 k=8 f=2048  dropless, Zipf gate bias
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass(frozen=True)
class MoEConfig:
    name: str
    T: int            # tokens of the whole EP group per layer call (b*s)
    d: int            # hidden size d_model
    E: int            # routed experts
    k: int            # top-k
    f: int            # expert FFN width d_ffn^MoE
    cf: float         # capacity factor; <= 0 means dropless
    E_s: int = 0      # shared experts (each width f)
    zipf_s: float = 0.0   # Zipf gate-bias strength (0 = none)

    def T_r(self, ep: int) -> int:
        return self.T // ep


CONFIGS = {
    "tiny": MoEConfig("tiny", T=256, d=64, E=8, k=2, f=128, cf=1.25),
    "mixtral": MoEConfig("mixtral", T=8192, d=4096, E=8, k=2, f=14336, cf=1.25),
    "dsmoe": MoEConfig("dsmoe", T=16384, d=2048, E=64, k=6, f=1408, cf=1.25, E_s=2),
    "dsv3": MoEConfig("dsv3", T=32768, d=7168, E=256, k=8, f=2048, cf=0.0, zipf_s=1.0),
    # profiling proxy (not a BASELINE config): one balanced EP=4 rank of dsv3 on one GPU --
    # 64 experts x ~1024 rows, d=7168, f=2048
    "dsv3_slice": MoEConfig("dsv3_slice", T=8192, d=7168, E=64, k=8, f=2048, cf=0.0),
}

SEED_X = 1
SEED_DY = 2
SEED_WR = 3
SEED_EXPERT0 = 100
SEED_SHARED0 = 10000
SEED_ZIPF = 1234


def _randn(shape, seed, std, device, dtype=torch.bfloat16):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t.to(dtype)


def tokens(cfg: MoEConfig, device="cpu", T: int | None = None, seed: int = SEED_X):
    """x [T, d] ~ N(0,1) in bf16; global tokens, sharded by rows across EP ranks."""
    return _randn((T or cfg.T, cfg.d), seed, 1.0, device)


def grad_output(cfg: MoEConfig, device="cpu", T: int | None = None, seed: int = SEED_DY):
    """dy [T, d] ~ N(0,1) in bf16."""
    return _randn((T or cfg.T, cfg.d), seed, 1.0, device)


def router_weight(cfg: MoEConfig, device="cpu"):
    """W_r stored as [E, d] (row e = the router column of expert e), N(0, 1/d) in bf16,
    so that the logits x.W_r are ~N(0,1)."""
    return _randn((cfg.E, cfg.d), SEED_WR, 1.0 / math.sqrt(cfg.d), device)


def expert_weights(cfg: MoEConfig, experts, device="cpu", width: int | None = None,
                   seed0: int = SEED_EXPERT0):
    """SwiGLU weights of the given global expert ids in the kernel layout:

    * ``w_gu``   [n, 2f, d] bf16: rows 0..f-1 = W_gate^T, rows f..2f-1 = W_up^T
    * ``w_down`` [n, d, f]  bf16: W_down^T

    (paper notation W_gate, W_up in R^{d x f}, W_down in R^{f x d}).
    W_gate, W_up ~ N(0, 1/d); W_down ~ N(0, 1/f).  Expert e draws from seed
    ``seed0 + e`` so its weights do not depend on which rank owns it."""
    f = width or cfg.f
    experts = list(experts)
    w_gu = torch.empty((len(experts), 2 * f, cfg.d), dtype=torch.bfloat16, device=device)
    w_down = torch.empty((len(experts), cfg.d, f), dtype=torch.bfloat16, device=device)
    for i, e in enumerate(experts):
        g = torch.Generator(device=device)
        g.manual_seed(seed0 + e)
        w_gu[i] = (torch.randn((2 * f, cfg.d), generator=g, device=device)
                   * (1.0 / math.sqrt(cfg.d))).to(torch.bfloat16)
        w_down[i] = (torch.randn((cfg.d, f), generator=g, device=device)
                     * (1.0 / math.sqrt(f))).to(torch.bfloat16)
    return w_gu, w_down


def shared_weights(cfg: MoEConfig, device="cpu"):
    """The E_s shared experts as ONE SwiGLU of width E_s*f (unweighted sum of
    E_s experts of width f == one expert of concatenated width)."""
    if cfg.E_s == 0:
        return None, None
    fs = cfg.E_s * cfg.f
    w_gu, w_down = expert_weights(cfg, [0], device=device, width=fs, seed0=SEED_SHARED0)
    return w_gu[0], w_down[0]


def zipf_bias(cfg: MoEConfig, s: float | None = None, permuted: bool = True):
    """Additive fp32 gate bias b_e = -s*ln(1+pi(e)), pi a seeded permutation of [0,E)
    (SURVEY.md §8(c) c.3-13).  Returns None when the config has no Zipf skew."""
    s = cfg.zipf_s if s is None else s
    if s == 0.0:
        return None
    g = torch.Generator()
    g.manual_seed(SEED_ZIPF)
    pi = torch.randperm(cfg.E, generator=g) if permuted else torch.arange(cfg.E)
    return (-s * torch.log1p(pi.to(torch.float64))).to(torch.float32)


def balanced_logits(T_r: int, E: int, k: int, ep_rank: int = 0):
    """The balanced fixture l[t,e] = -((e - k*t_g) mod E) (integers, exact in fp32):
    token t_g's top-k are experts k*t_g .. k*t_g+k-1 (mod E), so every expert gets
    exactly k*T_r/E rows per source rank when E | k*T_r."""
    t_g = torch.arange(T_r, dtype=torch.int64) + ep_rank * T_r
    e = torch.arange(E, dtype=torch.int64)
    return (-((e[None, :] - k * t_g[:, None]) % E)).to(torch.float32)


def drop_priority_logits(T_r: int, E: int):
    """Drop-priority fixture: every token picks experts {0,1};
    expert 0 is slot 0 for odd t and slot 1 for even t; the rest are -2-e."""
    L = torch.empty((T_r, E), dtype=torch.float32)
    L[:] = -2.0 - torch.arange(E, dtype=torch.float32)[None, :]
    t = torch.arange(T_r)
    odd = (t % 2) == 1
    L[:, 0] = torch.where(odd, 0.0, -1.0)
    L[:, 1] = torch.where(odd, -1.0, 0.0)
    return L


def random_logits(T: int, E: int, seed: int = 7, device="cpu"):
    """fp32 N(0,1) logits (the router's output scale), for routing-only tests."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn((T, E), generator=g, device=device, dtype=torch.float32)

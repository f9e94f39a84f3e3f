"""Seeded synthetic Q/K/V/dO tensors (INPUT GENERATOR ONLY — no attention arithmetic).

Values ~ N(0, 1) drawn in fp32 with one seed per (base, tensor, batch, head) so that
sharding heads across ranks never changes the data, then rounded
to bf16 (round-to-nearest-even, torch's cast).  Layout ``[B, N, H, d]`` contiguous,
the ABI layout of include/flashmask.h.
"""
from __future__ import annotations

import torch

TENSOR_IDS = {"q": 0, "k": 1, "v": 2, "do": 3}


def head_seed(base: int, name: str, b: int, h: int) -> int:
    return (((base * 1000003 + TENSOR_IDS[name]) * 10007 + b) * 1009 + h) & 0x7FFFFFFF


def make_tensor(name: str, B: int, N: int, H: int, d: int, base: int = 0,
                heads: range | None = None, dtype=torch.bfloat16) -> torch.Tensor:
    """CPU tensor [B, N, len(heads), d]; head slot i holds global head heads[i]."""
    heads = range(H) if heads is None else heads
    out = torch.empty(B, N, len(heads), d, dtype=dtype)
    g = torch.Generator()
    for b in range(B):
        for i, h in enumerate(heads):
            g.manual_seed(head_seed(base, name, b, h))
            out[b, :, i, :] = torch.randn(N, d, generator=g, dtype=torch.float32).to(dtype)
    return out


def make_qkv(B: int, N: int, H: int, d: int, base: int = 0, heads=None, with_do=True):
    names = ["q", "k", "v"] + (["do"] if with_do else [])
    return {n: make_tensor(n, B, N, H, d, base, heads) for n in names}


def make_device_tensor(name: str, B: int, N: int, H: int, d: int, base: int, device) -> torch.Tensor:
    """Large-shape variant for timing runs: one seeded device draw per tensor (Philox on the
    device), bf16.  Parity tests use ``make_tensor`` (per-head seeds on the CPU)."""
    g = torch.Generator(device=device)
    g.manual_seed(head_seed(base, name, 0, 0))
    x = torch.randn(B, N, H, d, generator=g, device=device, dtype=torch.float32)
    return x.to(torch.bfloat16)

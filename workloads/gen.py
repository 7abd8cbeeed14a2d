"""Seeded value generator for the synthetic checkpoint state.

Distributions mimic trained mixed-precision Adam state:
  master     ~ N(0, 0.02)  fp32   (GPT-3 init std)
  param      = bf16_RNE(master)   (the 16-bit model copy of the master weight)
  grad       ~ N(0, 1e-3)  bf16
  exp_avg    ~ N(0, 1e-4)  fp32
  exp_avg_sq = |N(0, 1e-6)| fp32
  randn      ~ N(0, 1)     in the Spec's dtype (C1 tiny tensors)
Full-entropy mantissas keep storage-level compression from flattering the
bandwidth numbers. Tensor i is drawn from torch.Generator seeded
SEED_BASE + Spec.gen_id (rank-local Specs already carry a rank offset).
Generation runs on any torch device; values differ between the CPU and CUDA
generators, so parity tests always hand the oracle the bytes of the exact
tensors the GPU path checkpoints (copied to host with torch, not our kernels).
"""
from __future__ import annotations

import torch

SEED_BASE = 0xFA572406

_TORCH_DTYPE = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16,
                "f64": torch.float64, "i64": torch.int64, "i32": torch.int32,
                "u8": torch.uint8}
_STD = {"master": 0.02, "param": 0.02, "grad": 1e-3, "exp_avg": 1e-4,
        "exp_avg_sq": 1e-6, "randn": 1.0}


def torch_dtype(dt: str):
    return _TORCH_DTYPE[dt]


def make_tensor(spec, device="cpu", seed_base: int = SEED_BASE) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed_base + int(spec.gen_id))
    dt = _TORCH_DTYPE[spec.dtype]
    if spec.numel == 0:
        return torch.empty(spec.shape, dtype=dt, device=device)
    if dt in (torch.int64, torch.int32, torch.uint8):
        hi = 256 if dt == torch.uint8 else 1 << 30
        return torch.randint(0, hi, spec.shape, generator=g, dtype=dt, device=device)
    x = torch.randn(spec.shape, generator=g, dtype=torch.float32, device=device)
    x.mul_(_STD[spec.gen])
    if spec.gen == "exp_avg_sq":
        x.abs_()
    return x.to(dt)


def make_state(specs, device="cpu", seed_base: int = SEED_BASE):
    """[(Spec, tensor)] in Spec order; each tensor is a fresh contiguous allocation."""
    return [(s, make_tensor(s, device, seed_base)) for s in specs]

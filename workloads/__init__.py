"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This package holds ONLY input generation: tensor shapes of the paper's GPT-3 /
MoE models (§5.2 Table `tb:gpt-setup`) and seeded random
values with the distributions of mixed-precision Adam state.
It contains none of the checkpoint method's arithmetic (no layout, no offsets,
no partitioning) so that the oracle (`oracle/`) and the CUDA path
(`paper_2406_13768_b200/`) can both consume it without sharing method code.
"""
from .shapes import (  # noqa: F401
    CONFIGS, Spec, config_specs, gpt3_tensors, gpt3_param_count, moe_tensors,
    tiny_tensors, state_bytes,
)
from .gen import make_tensor, make_state, SEED_BASE  # noqa: F401

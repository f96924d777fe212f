"""Seeded synthetic inputs shaped like the paper's workloads (configs 1-5).

Shared by the oracle tests and the GPU path; holds none of the method's
arithmetic (it only *prints* binary64 values as decimal text).  See
DESIGN.md "Inputs" for the recipes and csrc/fpgen.c for the C generator.
"""
from .gen import Workload, generate, CONFIG_N, CONFIG_SEP_MASK

__all__ = ["Workload", "generate", "CONFIG_N", "CONFIG_SEP_MASK"]

"""B200-native SymPhase sampling hot path (arXiv 2311.03906).

circuit text -> native symbolic pass (M_sym + channel table) -> fused sm_100a
sampler (Philox draws + GF(2) product + bit-packed records). See DESIGN.md.
"""
from .sampler import (InitResult, Sampler, pack_bits, parse_and_initialize, run_initialization,
                      unpack_bits)
from . import circuits

__all__ = ["InitResult", "Sampler", "pack_bits", "parse_and_initialize", "run_initialization",
           "unpack_bits", "circuits"]

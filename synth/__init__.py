"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no slot map, no attention):
it only draws request lengths, RT/BE classes, physical block assignments
(a stand-in for the host scheduler's FindBlock/FindPreemptBlock output) and
bf16 values from a counter-based hash that has identical numpy and torch
implementations.  Both the CPU oracle and the CUDA path consume what it
produces; neither side imports the other.
"""
from .workload import (CONFIGS, Shape, Layout, draw_lengths, build_layout, build_general_layout,
                       make_case,
                       Case, shard_heads)
from .values import (key32, hash_bf16_np, hash_bf16_torch, dense_kv_np, q_np,
                     dense_kv_torch, q_torch, q_rows_np, q_rows_torch, BF16_NAN)

__all__ = [
    "CONFIGS", "Shape", "Layout", "draw_lengths", "build_layout", "build_general_layout", "make_case", "Case",
    "shard_heads", "key32", "hash_bf16_np", "hash_bf16_torch", "dense_kv_np", "q_np",
    "dense_kv_torch", "q_torch", "q_rows_np", "q_rows_torch", "BF16_NAN",
]

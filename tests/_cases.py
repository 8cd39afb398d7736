"""Test-side helpers: materialise a synth.Case on the host through the ORACLE.

Used by CPU oracle pins and by the GPU parity tests (as the expected side).
Never imports the product package.
"""
from __future__ import annotations

import math

import numpy as np

import oracle
from synth import dense_kv_np, q_np
from synth.values import BF16_NAN


def dense_case(case, kv_heads=None, q_heads=None):
    """Per-request dense K/V (uint16 [L][H][d]) and q (uint16 [B][Hq][d])."""
    sh, lay = case.shape, case.layout
    kv_heads = list(range(sh.num_kv_heads)) if kv_heads is None else list(kv_heads)
    q_heads = list(range(sh.num_q_heads)) if q_heads is None else list(q_heads)
    ks, vs = [], []
    for r in range(lay.batch):
        k, v = dense_kv_np(case.seed, case.layer, r, int(lay.lens[r]), kv_heads, sh.head_dim,
                           sh.num_kv_heads)
        ks.append(k)
        vs.append(v)
    q = np.stack([q_np(case.seed, case.layer, r, q_heads, sh.head_dim, case.q_scale_log2)
                  for r in range(lay.batch)]) if lay.batch else np.zeros((0, len(q_heads), sh.head_dim), np.uint16)
    return ks, vs, q


def ragged(ks, vs, lens, before):
    """Concatenate tokens [before[r], lens[r]) of every request -> (k_new, v_new, cu_new)."""
    cu = [0]
    kn, vn = [], []
    for r in range(len(lens)):
        kn.append(ks[r][before[r]:lens[r]])
        vn.append(vs[r][before[r]:lens[r]])
        cu.append(cu[-1] + int(lens[r]) - int(before[r]))
    H, d = ks[0].shape[1:] if ks else (1, 1)
    k_new = np.concatenate(kn) if kn else np.zeros((0, H, d), np.uint16)
    v_new = np.concatenate(vn) if vn else np.zeros((0, H, d), np.uint16)
    return k_new, v_new, np.asarray(cu, dtype=np.int32)


def oracle_pool(case, ks, vs, n_heads, fill=BF16_NAN, per_request_dirs=False):
    """Fill a host pool by appending every resident token through the oracle."""
    sh, lay = case.shape, case.layout
    K, V = oracle.new_pool(lay.num_blocks, n_heads, sh.block_size, sh.head_dim, fill)
    before = np.zeros(lay.batch, dtype=np.int32)
    k_new, v_new, cu = ragged(ks, vs, lay.lens, before)
    dirs = lay.dirs_per_request if per_request_dirs else lay.dirs
    sm = oracle.append(K, V, lay.block_tables, dirs, before, cu, k_new, v_new)
    return K, V, sm


def default_scale(d):
    return 1.0 / math.sqrt(d)

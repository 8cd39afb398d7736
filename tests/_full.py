"""Full-size parity harness: a BASELINE-size batch on the GPU, every output element
(B x H_q x d) and -- for the fused step -- every pool byte checked against the oracle.

The oracle side is built only from synth/ values and oracle/ calls (no input or
expected value comes from the CUDA path); the GPU side generates the same values
with the bit-identical torch twin of the counter hash.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case, dense_kv_np, dense_kv_torch, q_np, q_torch
from synth.values import BF16_NAN
from synth.workload import shard_heads

MAX_ABS, MEAN_ABS = 2e-2, 2e-3
DEV = "cuda"


def _fill(t, bits):
    t.view(torch.int16).fill_(int(np.uint16(bits).view(np.int16)))


def run_full(cfg, tp=1, rank=0, seed=0, mode="step", pdl=True, planned=False, spare_blocks=3,
             general=False, check_pool=True, chunk=32, repeat=1):
    """Returns (gpu out [B][Hq][d] float64, oracle out, per-request max-abs error)."""
    sh = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    case = make_case(sh, seed, spare_blocks=spare_blocks, general=general)
    lay = case.layout
    kv_heads, q_heads = shard_heads(sh, tp, rank)
    Hl, d, bs, B = len(kv_heads), sh.head_dim, sh.block_size, lay.batch
    gm_np = dict(fills=lay.fills, num_entries=lay.num_entries) if general else {}
    resident = lay.lens - (1 if mode == "step" else 0)
    # ---- GPU side
    pool = bkv.KVPool.empty(lay.num_blocks, Hl, bs, d, DEV)
    _fill(pool.k, BF16_NAN)
    _fill(pool.v, BF16_NAN)
    bt = torch.from_numpy(lay.block_tables).to(DEV)
    dirs = torch.from_numpy(lay.dirs).to(DEV)
    lens = torch.from_numpy(lay.lens.astype(np.int32)).to(DEV)
    gm = dict(fills=torch.from_numpy(lay.fills).to(DEV), num_entries=torch.from_numpy(lay.num_entries).to(DEV)) \
        if general else {}
    last_k, last_v = [], []
    for r0 in range(0, B, chunk):
        rs = list(range(r0, min(B, r0 + chunk)))
        kk, vv = zip(*[dense_kv_torch(case.seed, 0, r, int(lay.lens[r]), kv_heads, d, sh.num_kv_heads, DEV)
                       for r in rs])
        last_k += [k[-1] for k in kk]
        last_v += [v[-1] for v in vv]
        kn = torch.cat([k[:resident[r]] for k, r in zip(kk, rs)])
        vn = torch.cat([v[:resident[r]] for v, r in zip(vv, rs)])
        cu = torch.tensor(np.concatenate([[0], np.cumsum(resident[rs])]), dtype=torch.int32, device=DEV)
        sub = {k: v[r0:r0 + len(rs)].contiguous() for k, v in gm.items()}
        bkv.kv_append(pool, bt[r0:r0 + len(rs)].contiguous(), dirs[r0:r0 + len(rs)].contiguous(),
                      torch.zeros(len(rs), dtype=torch.int32, device=DEV), cu,
                      kn, vn, **sub)
    q = torch.stack([q_torch(case.seed, 0, r, q_heads, d, DEV) for r in range(B)])
    kl = torch.stack(last_k).contiguous()
    vl = torch.stack(last_v).contiguous()
    scale = 1.0 / math.sqrt(d)
    plan = None
    if planned:
        plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, len(q_heads),
                               fills_host=lay.fills if general else None,
                               num_entries_host=lay.num_entries if general else None)
    outs = []
    for it in range(repeat):   # (a repeated fused step re-writes the same token: idempotent)
        if planned:
            o = bkv.decode_planned(pool, bt, dirs, lens, plan, q, k_new=kl if mode == "step" else None,
                                   v_new=vl if mode == "step" else None, pdl=pdl, **gm)
        elif mode == "step":
            o = bkv.decode_step(pool, bt, dirs, lens, kl, vl, q, pdl=pdl, **gm)
        else:
            o = bkv.paged_decode_attention(pool, bt, dirs, lens, q, pdl=pdl, **gm)
        outs.append(o.clone())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16)), "run-to-run bitwise determinism"
    got = outs[0].float().cpu().numpy().astype(np.float64)
    # ---- oracle side: every resident token appended through the oracle, attention over all rows
    K, V = oracle.new_pool(lay.num_blocks, Hl, bs, d, BF16_NAN)
    for r0 in range(0, B, chunk):
        rs = list(range(r0, min(B, r0 + chunk)))
        kv = [dense_kv_np(case.seed, 0, r, int(lay.lens[r]), kv_heads, d, sh.num_kv_heads) for r in rs]
        kn = np.concatenate([k for k, _ in kv])
        vn = np.concatenate([v for _, v in kv])
        cu = np.concatenate([[0], np.cumsum(lay.lens[rs])]).astype(np.int32)
        sub = {k: np.ascontiguousarray(v[r0:r0 + len(rs)]) for k, v in gm_np.items()}
        oracle.append(K, V, np.ascontiguousarray(lay.block_tables[r0:r0 + len(rs)]),
                      np.ascontiguousarray(lay.dirs[r0:r0 + len(rs)]), np.zeros(len(rs), np.int32), cu, kn, vn,
                      **sub)
    qn = np.stack([q_np(case.seed, 0, r, q_heads, d) for r in range(B)])
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, qn, scale, **gm_np)
    if mode == "step" and check_pool:   # the fused append at full size: every pool byte
        gk = pool.k.view(torch.int16).cpu().numpy().view(np.uint16)
        gv = pool.v.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(gk, K) and np.array_equal(gv, V), "fused append: pool differs from the oracle"
    assert np.isfinite(got).all()
    err = np.abs(got - ref)
    per_req = err.reshape(B, -1).max(1)
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (sh.name, tp, rank, err.max(), err.mean(),
                                                             int(per_req.argmax()))
    return got, ref, per_req

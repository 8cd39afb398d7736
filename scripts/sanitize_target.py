"""Small driver for compute-sanitizer: append + decode attention (+ split merge)
+ checkpoint/restore on tiny MHA and GQA configs, both directions, shared tails."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BKV_MIN_SPLIT", "1")         # force splits so merge_kernel runs
os.environ.setdefault("BKV_UNITS_PER_WARP", "64")
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from synth import make_case
from synth.workload import Shape
from tests._cases import dense_case, ragged

def g(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)

for sh in (Shape("s1", 4, 4, 64, 16, 8, 0.5, "uniform", 300, 1, 1, uniform_max=300),
           Shape("s2", 8, 1, 128, 16, 8, 0.5, "uniform", 300, 1, 1, uniform_max=300),
           Shape("s3", 16, 2, 128, 32, 6, 0.5, "uniform", 300, 1, 1, uniform_max=300)):
    case = make_case(sh, 1)
    lay = case.layout
    ks, vs, q = dense_case(case)
    pool = bkv.KVPool.empty(lay.num_blocks, sh.num_kv_heads, sh.block_size, sh.head_dim)
    pool.k.zero_(); pool.v.zero_()
    kn, vn, cu = ragged(ks, vs, lay.lens, np.zeros(lay.batch, np.int64))
    bt = torch.from_numpy(lay.block_tables).cuda(); dirs = torch.from_numpy(lay.dirs).cuda()
    sm = torch.zeros(kn.shape[0], dtype=torch.int64, device="cuda")
    bkv.kv_append(pool, bt, dirs, torch.zeros(lay.batch, dtype=torch.int32, device="cuda"),
                  torch.from_numpy(cu).cuda(), g(kn), g(vn), slot_mapping=sm)
    for pdl in (False, True):
        out = bkv.paged_decode_attention(pool, bt, dirs, torch.from_numpy(lay.lens).cuda(), g(q), pdl=pdl)
    os.environ["BKV_STREAMK"] = "2"   # stream-K plan (rows cut across warp ranges) on the same case
    bkv.reload_dev_switches()
    out = bkv.paged_decode_attention(pool, bt, dirs, torch.from_numpy(lay.lens).cuda(), g(q), pdl=True)
    os.environ["BKV_STREAMK"] = "1"
    bkv.reload_dev_switches()
    ck, cv = bkv.kv_checkpoint(pool, sm[:17])
    bkv.kv_restore(pool, sm[:17], ck, cv)
    torch.cuda.synchronize()
    print(sh.name, "ok", float(out.float().abs().mean()))

# round r01c additions: general maps (f3), fused decode step, fused checkpoint (f1), prefill (f4)
from tests.test_prefill_oracle import query_counts
from synth import q_rows_np
for sh in (Shape("g1", 4, 4, 64, 16, 8, 0.5, "uniform", 300, 1, 1, uniform_max=300),
           Shape("g2", 8, 1, 128, 32, 8, 0.5, "uniform", 300, 1, 1, uniform_max=300)):
    case = make_case(sh, 2, general=True, share_prob=1.0)
    lay = case.layout
    ks, vs, q = dense_case(case)
    pool = bkv.KVPool.empty(lay.num_blocks, sh.num_kv_heads, sh.block_size, sh.head_dim)
    pool.k.zero_(); pool.v.zero_()
    bt = torch.from_numpy(lay.block_tables).cuda(); dirs = torch.from_numpy(lay.dirs).cuda()
    fills = torch.from_numpy(lay.fills).cuda(); nent = torch.from_numpy(lay.num_entries).cuda()
    before = np.maximum(lay.lens - 1, 0).astype(np.int32)
    kn, vn, cu = ragged(ks, vs, before, np.zeros(lay.batch, np.int64))
    bkv.kv_append(pool, bt, dirs, torch.zeros(lay.batch, dtype=torch.int32, device="cuda"),
                  torch.from_numpy(cu).cuda(), g(kn), g(vn), fills=fills, num_entries=nent)
    kd = np.stack([ks[r][lay.lens[r] - 1] for r in range(lay.batch)])
    vd = np.stack([vs[r][lay.lens[r] - 1] for r in range(lay.batch)])
    lens = torch.from_numpy(lay.lens).cuda()
    out = bkv.decode_step(pool, bt, dirs, lens, g(kd), g(vd), g(q), fills=fills, num_entries=nent)
    out2 = bkv.paged_decode_attention(pool, bt, dirs, lens, g(q), fills=fills, num_entries=nent)
    n = query_counts(lay.lens, np.random.default_rng(0))
    qp = np.concatenate([q_rows_np(0, 0, r, int(n[r]), range(sh.num_q_heads), sh.head_dim, sh.num_q_heads)
                         for r in range(lay.batch)])
    cuq = torch.from_numpy(np.concatenate([[0], np.cumsum(n)]).astype(np.int32)).cuda()
    op = bkv.paged_prefill_attention(pool, bt, dirs, lens, cuq, g(qp), fills=fills, num_entries=nent)
    # fused lazy checkpoint: every new token evicts into its own checkpoint row
    ev = torch.arange(lay.batch, dtype=torch.int32, device="cuda")
    ckk = torch.empty((lay.batch, sh.num_kv_heads, sh.head_dim), dtype=torch.bfloat16, device="cuda")
    ckv = torch.empty_like(ckk)
    bkv.kv_append_checkpoint(pool, bt, dirs, torch.from_numpy(before).cuda(),
                             torch.arange(lay.batch + 1, dtype=torch.int32, device="cuda"), g(kd), g(vd),
                             ev, ckk, ckv, fills=fills, num_entries=nent)
    torch.cuda.synchronize()
    print(sh.name, "general ok", float(out.float().abs().mean()), float(op.float().abs().mean()))

# round r02: the planned decode (host plan, one decode kernel + cross-CTA merge kernel per layer),
# both cross-CTA merge modes, fused step, early KV tiles, peers, on small and TP-shard shapes
from synth import CONFIGS
from synth.workload import shard_heads
for cfg, tp in (("tiny_gqa", 1), ("llama70b", 8), ("opt13b", 8)):
    sh = CONFIGS[cfg]
    lay = make_case(cfg, 3).layout
    kvh, qh = shard_heads(sh, tp, 0)
    H, Hq, d = len(kvh), len(qh), sh.head_dim
    pool = bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16),
                      torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16))
    bt = torch.from_numpy(lay.block_tables).cuda(); dirs = torch.from_numpy(lay.dirs).cuda()
    lens = torch.from_numpy(lay.lens).cuda()
    qd = torch.randn(lay.batch, Hq, d, device="cuda").to(torch.bfloat16)
    kd = torch.randn(lay.batch, H, d, device="cuda").to(torch.bfloat16)
    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, Hq)
    peer = torch.empty_like(qd)
    o1 = bkv.decode_planned(pool, bt, dirs, lens, plan, qd, k_new=kd, v_new=kd, pdl=True, kv_early=True)
    o2 = bkv.decode_planned(pool, bt, dirs, lens, plan, qd, peer_outs=[peer])
    torch.cuda.synchronize()
    print(cfg, tp, "planned ok", float(o1.float().abs().mean()), float(o2.float().abs().mean()))

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
    ck, cv = bkv.kv_checkpoint(pool, sm[:17])
    bkv.kv_restore(pool, sm[:17], ck, cv)
    torch.cuda.synchronize()
    print(sh.name, "ok", float(out.float().abs().mean()))

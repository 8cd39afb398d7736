"""Small eager driver for ncu: n fused planned decode steps (bkv_decode_planned) of one shard."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case
from synth.workload import shard_heads

cfg, tp = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
sh = CONFIGS[cfg]; lay = make_case(cfg, 0).layout
kvh, qh = shard_heads(sh, tp, 0); H, Hq, d, B = len(kvh), len(qh), sh.head_dim, lay.batch
pool = bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16),
                  torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16))
bt = torch.from_numpy(lay.block_tables).cuda(); dirs = torch.from_numpy(lay.dirs).cuda()
lens = torch.from_numpy(lay.lens).cuda(); q = torch.randn(B, Hq, d, device="cuda").to(torch.bfloat16)
kn = torch.randn(B, H, d, device="cuda").to(torch.bfloat16)
vn = torch.randn(B, H, d, device="cuda").to(torch.bfloat16)
plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, Hq)
for _ in range(n):
    bkv.decode_planned(pool, bt, dirs, lens, plan, q, k_new=kn, v_new=vn, pdl=True, kv_early=True)
torch.cuda.synchronize()
print("plan P", plan.header["P"])

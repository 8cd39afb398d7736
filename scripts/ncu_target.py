"""Small eager driver for ncu: a few decode-attention launches of one config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case
from synth.workload import shard_heads

cfg, tp = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
sh = CONFIGS[cfg]; lay = make_case(cfg, 0).layout
kvh, qh = shard_heads(sh, tp, 0); H, Hq, d = len(kvh), len(qh), sh.head_dim
pool = bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16),
                  torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16))
bt = torch.from_numpy(lay.block_tables).cuda(); dirs = torch.from_numpy(lay.dirs).cuda()
lens = torch.from_numpy(lay.lens).cuda(); q = torch.randn(lay.batch, Hq, d, device="cuda").to(torch.bfloat16)
B = lay.batch
kn = torch.randn(B, H, d, device="cuda").to(torch.bfloat16)
before = torch.from_numpy((lay.lens - 1).astype(np.int32)).cuda(); cu = torch.arange(B + 1, dtype=torch.int32, device="cuda")
for _ in range(n):
    bkv.kv_append(pool, bt, dirs, before, cu, kn, kn)
    bkv.paged_decode_attention(pool, bt, dirs, lens, q)
torch.cuda.synchronize()
print("algorithmic bytes per attention launch:", float(lay.lens.sum()) * 4 * H * d + 4 * B * Hq * d)

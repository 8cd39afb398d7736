"""Dev: timeline of the planned decode kernel over consecutive layers (CUDA graph, PDL).

Needs a trace build:  BKV_BUILD_TRACE=1 python paper_2504_09590_b200/build.py --force
    BKV_TRACE=4 python scripts/trace_planned.py llama70b 8 [layers]
Each layer gets its own workspace (so its trace region survives); per warp the kernel
stamps %globaltimer at: 0 entry, 1 pre-wait reads, 2 grid wait, 3 first tile,
4 streaming done, 5 CTA barrier, 6 merges done.
"""
import os
import sys

os.environ.setdefault("BKV_TRACE", "8")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case
from synth.workload import shard_heads

cfg, tp = sys.argv[1], int(sys.argv[2])
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 6
mode = sys.argv[4] if len(sys.argv) > 4 else "step"
sh = CONFIGS[cfg]
lay = make_case(cfg, 0).layout
kvh, qh = shard_heads(sh, tp, 0)
H, Hq, d = len(kvh), len(qh), sh.head_dim
dev = "cuda"
pools = [bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device=dev).to(torch.bfloat16),
                    torch.randn(lay.num_blocks, H, sh.block_size, d, device=dev).to(torch.bfloat16)) for _ in range(nl)]
bt = torch.from_numpy(lay.block_tables).to(dev)
dirs = torch.from_numpy(lay.dirs).to(dev)
lens = torch.from_numpy(lay.lens).to(dev)
q = torch.randn(lay.batch, Hq, d, device=dev).to(torch.bfloat16)
kn = torch.randn(lay.batch, H, d, device=dev).to(torch.bfloat16)
vn = torch.randn(lay.batch, H, d, device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
need = bkv.decode_workspace_size(lay.batch, Hq, H, d)
wss = [torch.zeros(need, dtype=torch.uint8, device=dev) for _ in range(nl)]
plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pools[0], Hq)
hd = plan.header
W = hd["grid"] * hd["warps"]
tr_bytes = W * 16 * 8
start = need - ((W * int(os.environ["BKV_TRACE"]) * 16 + 255) // 256 * 256)


def body():
    for l in range(nl):
        if mode in ("step", "early"):
            bkv.decode_planned(pools[l], bt, dirs, lens, plan, q, k_new=kn, v_new=vn, out=out, ws=wss[l], pdl=True,
                               kv_early=mode == "early")
        else:
            bkv.decode_planned(pools[l], bt, dirs, lens, plan, q, out=out, ws=wss[l], pdl=True)


body()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    body()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for w in wss:
    w[start:start + tr_bytes].zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"{cfg} tp{tp} {mode}: graph of {nl} layers {e0.elapsed_time(e1) * 1e3 / nl:.1f} us/layer "
      f"(P {hd['P']} blocks/warp, {hd['n_segs']} segs, {hd['n_tasks']} tasks, max pieces {hd['max_pieces']})")
T = np.stack([w[start:start + tr_bytes].view(torch.int64).cpu().numpy().reshape(W, 16) for w in wss])   # [layer][warp][k]
t0 = T[0, :, 0][T[0, :, 0] > 0].min()
T = np.where(T > 0, T - t0, -1) / 1e3    # us
names = ["entry", "prewait", "gridwait", "first", "stream_end", "barrier", "merged"]
for l in range(nl):
    row = []
    for k, n in enumerate(names):
        v = T[l, :, k]
        v = v[v >= 0]
        row.append(f"{n} {np.median(v):6.2f}/{v.max():6.2f}" if v.size else f"{n} -")
    print(f"  L{l}: " + "  ".join(row))
# busy per warp: streaming duration distribution of one middle layer
l = nl // 2
s = T[l, :, 4] - T[l, :, 3]
print(f"  L{l} per-warp streaming (first tile -> done): p10 {np.percentile(s, 10):.2f} p50 {np.median(s):.2f} "
      f"p90 {np.percentile(s, 90):.2f} max {s.max():.2f} us; merges (barrier -> merged) max "
      f"{(T[l, :, 6] - T[l, :, 5]).max():.2f} us; first tile after wait p50 {np.median(T[l, :, 3] - T[l, :, 2]):.2f}")
for a, b in ((4, 5), (5, 6)):
    ok = (T[l, :, a] >= 0) & (T[l, :, b] >= 0)
    dd = T[l, ok, b] - T[l, ok, a]
    if dd.size:
        print(f"  {names[a]} -> {names[b]}: n {dd.size} p50 {np.median(dd):.2f} p90 {np.percentile(dd, 90):.2f} max {dd.max():.2f} us")
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
np.savez(os.path.join(out_dir, f"trace_{cfg}_tp{tp}_{mode}.npz"), T=T, warps=hd["warps"], grid=hd["grid"])


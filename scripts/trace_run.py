"""Dev: run one decode launch with BKV_TRACE and summarise the per-warp timeline.

Needs a trace build: BKV_BUILD_TRACE=1 python paper_2504_09590_b200/build.py --force
"""
import os, sys
os.environ.setdefault("BKV_TRACE", "64")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case
from synth.workload import shard_heads
cfg, tp = sys.argv[1], int(sys.argv[2])
sh = CONFIGS[cfg]; lay = make_case(cfg, 0).layout
kvh, qh = shard_heads(sh, tp, 0); H, Hq, d = len(kvh), len(qh), sh.head_dim
pools = [bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16),
                    torch.randn(lay.num_blocks, H, sh.block_size, d, device="cuda").to(torch.bfloat16)) for _ in range(4)]
bt = torch.from_numpy(lay.block_tables).cuda(); dirs = torch.from_numpy(lay.dirs).cuda()
lens = torch.from_numpy(lay.lens).cuda(); q = torch.randn(lay.batch, Hq, d, device="cuda").to(torch.bfloat16)
ws = bkv.workspace(lay.batch, Hq, H, d)
cap = int(os.environ["BKV_TRACE"])
nw = 148 * int(os.environ.get("BKV_WARPS", "8" if Hq > H else "12"))
need = nw * cap * 16
total = bkv.decode_workspace_size(lay.batch, Hq, H, d)   # trace region = last up256(need) bytes
start = total - ((need + 255) // 256 * 256)
for p in pools[:3]: bkv.paged_decode_attention(p, bt, dirs, lens, q, ws=ws)
ws[start:start + need].zero_()
bkv.paged_decode_attention(pools[3], bt, dirs, lens, q, ws=ws)
torch.cuda.synchronize()
tr = ws[start:start + need].view(torch.int64).cpu().numpy().reshape(nw, cap, 2)
t = (tr[:, :, 0].astype(np.uint64) >> np.uint64(8)).astype(np.int64)
k = (tr[:, :, 0] & 0xFF)
valid = t > 0
t0 = t[valid].min()
tt = np.where(valid, t - t0, -1)
def col(kind):
    return np.where((k == kind) & valid, tt, -1)
start_k = col(0).max(1); plan_done = col(1).max(1); exit_ = col(6).max(1)
print(f"{cfg} tp{tp}: kernel span {tt.max()/1e3:.1f} us; prologue median {np.median(plan_done - start_k)/1e3:.2f} us; "
      f"warp start spread {np.ptp(start_k)/1e3:.2f} us; exit p50 {np.median(exit_)/1e3:.1f} max {exit_.max()/1e3:.1f} us")
# per unit: grab (2) -> first consume (3) -> end (4)
g2, g3, g4 = [], [], []
for w in range(nw):
    ev = {}
    for j in range(cap):
        if not valid[w, j]: continue
        ev.setdefault((k[w, j], tr[w, j, 1]), tt[w, j])
    for (kind, u), v in ev.items():
        if kind == 2 and (3, u) in ev and (4, u) in ev:
            g2.append(ev[(3, u)] - v); g3.append(ev[(4, u)] - ev[(3, u)]); g4.append(ev[(4, u)])
g2, g3 = np.array(g2), np.array(g3)
print(f"  units {len(g2)}: grab->first-data median {np.median(g2)/1e3:.2f} us p90 {np.percentile(g2,90)/1e3:.2f}; "
      f"first-data->end median {np.median(g3)/1e3:.2f} us p90 {np.percentile(g3,90)/1e3:.2f} max {g3.max()/1e3:.2f}")
busy = (exit_ - plan_done)
print(f"  units per warp: {np.bincount((col(4) >= 0).sum(1))[:8]}")

# per-warp cycle breakdown (kinds 8..13: wait, smem->reg, issue, math, end-of-unit, chunks)
vals = np.zeros((nw, 6))
for kk in range(6):
    sel = (k == 8 + kk) & valid
    vals[:, kk] = np.where(sel, tr[:, :, 1], 0).sum(1)
act = vals[:, 5] > 0
v = vals[act]
names = ["wait", "begin-unit", "consume", "issue", "end-unit"]
tot = v[:, :5].sum(1)
print("  per-warp cycles (active warps, median): " + ", ".join(f"{n} {np.median(v[:, i]):.0f}" for i, n in enumerate(names)) +
      f"; chunks {np.median(v[:, 5]):.0f}; per chunk: " + ", ".join(f"{n} {np.median(v[:, i] / np.maximum(v[:, 5], 1)):.0f}" for i, n in enumerate(names)))

# prologue clocks (kinds 16..20: after seq_lens loads, after the total reduction,
# after P, after the bucket scans, plan done -- cycles since kernel entry)
pro = []
for kk in range(16, 21):
    sel = (k == kk) & valid
    if sel.any():
        pro.append(np.median(tr[:, :, 1][sel]))
if pro:
    print("  prologue cycles since entry (median over warps): loads %.0f, reduce %.0f, P %.0f, scans %.0f, done %.0f" % tuple(pro))

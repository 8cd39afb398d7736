"""Dev: cycle accounting of the tcgen05 prefill kernel (needs a trace build:
BKV_BUILD_TRACE=1 python paper_2504_09590_b200/build.py --force)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from scripts.bench_prefill import setup
from synth import CONFIGS, make_case

cfg, tp = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("llama70b", 1)
shape = CONFIGS[cfg]
lay = make_case(shape, 0).layout
rng = np.random.default_rng(1)
be = np.flatnonzero(lay.is_be)
pre = rng.choice(be, size=min(16, be.size), replace=False)
n = np.zeros(lay.batch, np.int32)
n[pre] = lay.lens[pre]
fn, H, Hq, d = setup(shape, lay, tp, 2, n, 0)
L = bkv.lib()
L.bkv_dev_prefill_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(148 * 3 * 8, np.uint64)
fn(); torch.cuda.synchronize()
L.bkv_dev_prefill_prof(buf.ctypes.data, 1)
fn(); torch.cuda.synchronize()
rc = L.bkv_dev_prefill_prof(buf.ctypes.data, 1)
b = buf.reshape(148, 3, 8).astype(np.float64)
tiles = b[:, 0, 7].sum()
print(f"rc {rc}  key tiles (2 layers) {tiles:.0f}")
names = {0: ["meta bar", "full", "zero+walk", "s_full wait", "ld+mask+max+resc", "p_free wait", "exp+P store", "tiles"],
         1: ["meta bar", "full wait", "s_free wait", "S issue", "PV (p_full wait+issue)", "-", "-", "-"]}
it = b[:, 2, :].sum(0)
print(f"items {it[1]:.0f}  per CTA: kernel cycles {b[:, 2, 0].mean():.0f} (max {b[:, 2, 0].max():.0f}), tiles {tiles / 148:.1f}, items {it[1] / 148:.1f}")
print(f"softmax thread 0 per item: start->first tile {it[2] / max(it[1], 1):.0f}, epilogue {it[3] / max(it[1], 1):.0f}, "
      f"next-item search {it[4] / max(it[1], 1):.0f} cycles")
for role in (0, 1):
    tot = b[:, role, :7].sum(0)
    print(["softmax warp 0", "MMA lane"][role] + ": " + ", ".join(
        f"{names[role][i]} {tot[i] / max(tiles, 1):.0f}" for i in range(7 if role == 0 else 5)) + "  (cycles per tile)")

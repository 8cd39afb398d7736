"""Dev: event timeline of CTA 0 of the tcgen05 prefill kernel (trace build:
BKV_BUILD_TRACE=1 python paper_2504_09590_b200/build.py --force).  Prints the
events of a few steady-state work items, cycles relative to the first shown."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from scripts.bench_prefill import setup
from synth import CONFIGS, make_case

cfg, tp = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("llama70b", 1)
first, count = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (6, 2)
shape = CONFIGS[cfg]
lay = make_case(shape, 0).layout
rng = np.random.default_rng(1)
be = np.flatnonzero(lay.is_be)
pre = rng.choice(be, size=min(16, be.size), replace=False)
n = np.zeros(lay.batch, np.int32)
n[pre] = lay.lens[pre]
fn, H, Hq, d = setup(shape, lay, tp, 1, n, 0)
L = bkv.lib()
L.bkv_dev_prefill_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(2 * 12 * 2048, np.uint64)
fn(); torch.cuda.synchronize()
L.bkv_dev_prefill_trace(buf.ctypes.data, 1)
fn(); torch.cuda.synchronize()
cnt = L.bkv_dev_prefill_trace(buf.ctypes.data, 1)
ev = buf.reshape(-1, 2)
ev = ev[ev[:, 0] != 0]
cnt = len(ev)
ev = ev[np.argsort(ev[:, 0], kind="stable")]
names = {0: "P item start", 1: "P walk init+first tile", 2: "K Q issued", 3: "P stage free->TMA",
         15: "M s_free q0", 16: "M s_free q1", 17: "M p_full q0", 18: "M p_full q1", 10: "M meta", 11: "M full", 12: "M S issued", 13: "M PV(t-1) issued", 14: "M PV(last) issued",
         20: "S wait meta", 21: "S meta", 22: "S s_full", 23: "S P stored", 24: "S epi start", 25: "S epi p_free",
         26: "S epi done"}
# items: count softmax warp 0 "epi done" events
done = np.flatnonzero((ev[:, 1] & 0xffff) == 26)
print(f"events {cnt}, items done by warp 0: {len(done)}; total span {int(ev[-1, 0] - ev[0, 0])} cycles")
lo = done[first - 1] if first >= 1 else 0
hi = done[min(first + count - 1, len(done) - 1)]
t0 = int(ev[lo, 0])
for c, w in ev[lo:hi + 1]:
    w = int(w)
    print(f"{int(c) - t0:8d}  warp {(w >> 8) & 255:2d}  tile {w >> 16:4d}  {names.get(w & 255, w & 255)}")

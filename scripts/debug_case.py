"""Dev helper: per-(request, head) error of one geometry, optional env overrides."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_parity import _run_case
from synth import make_case
from synth.workload import Shape

def go(hq, hkv, d, bs, B=20, ctx=700, seed=None):
    sh = Shape("geo", hq, hkv, d, bs, B, 0.5, "uniform", ctx, 1, 1, uniform_max=ctx)
    case = make_case(sh, hq * 7 + bs if seed is None else seed, q_scale_log2=2)
    o, ref, _ = _run_case(case)
    err = np.abs(o.float().cpu().numpy() - ref)
    e_rh = err.max(axis=2)
    bad = np.argwhere(e_rh > 2e-2)
    print(f"hq{hq} hkv{hkv} d{d} bs{bs} env={ {k:v for k,v in os.environ.items() if k.startswith('BKV')} }: max {err.max():.3e} mean {err.mean():.3e} bad(r,h)={bad[:12].tolist()} n_bad={len(bad)}")
    if len(bad):
        L = case.layout.lens
        print("   lens of bad requests:", sorted(set(int(L[r]) for r, _ in bad)), " dirs:", sorted(set(int(case.layout.is_be[r]) for r,_ in bad)))

for spec in sys.argv[1:]:
    go(*[int(x) for x in spec.split(",")])

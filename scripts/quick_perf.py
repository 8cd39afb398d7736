"""Quick per-layer timing of decode attention (CUDA graph of all layers, CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case
from synth.workload import shard_heads

def run(cfg, tp=1, layers=8, iters=20, mode="attn"):
    sh = CONFIGS[cfg]; case = make_case(cfg, 0); lay = case.layout
    kvh, qh = shard_heads(sh, tp, 0); H = len(kvh); Hq = len(qh); d = sh.head_dim
    dev = "cuda"
    layers = max(layers, int(np.ceil(600e6 / (lay.lens.sum() * 4 * H * d))))   # >= 4.7x L2 rotating
    pools = [bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device=dev).to(torch.bfloat16),
                        torch.randn(lay.num_blocks, H, sh.block_size, d, device=dev).to(torch.bfloat16))
             for _ in range(layers)]
    bt = torch.from_numpy(lay.block_tables).to(dev); dirs = torch.from_numpy(lay.dirs).to(dev)
    lens = torch.from_numpy(lay.lens).to(dev)
    q = torch.randn(lay.batch, Hq, d, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws = bkv.workspace(lay.batch, Hq, H, d)
    kn = torch.randn(lay.batch, H, d, device=dev).to(torch.bfloat16)
    vn = torch.randn(lay.batch, H, d, device=dev).to(torch.bfloat16)
    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pools[0], Hq) if mode.startswith("planned") else None
    def body():
        for p in pools:
            if mode == "planned":
                bkv.decode_planned(p, bt, dirs, lens, plan, q, k_new=kn, v_new=vn, out=out, ws=ws, pdl=True)
            elif mode == "planned_early":
                bkv.decode_planned(p, bt, dirs, lens, plan, q, k_new=kn, v_new=vn, out=out, ws=ws, pdl=True,
                                   kv_early=True)
            elif mode == "planned_attn":
                bkv.decode_planned(p, bt, dirs, lens, plan, q, out=out, ws=ws, pdl=True)
            elif mode == "fused":
                bkv.decode_step(p, bt, dirs, lens, kn, vn, q, out=out, ws=ws, pdl=True)
            else:
                bkv.paged_decode_attention(p, bt, dirs, lens, q, out=out, ws=ws, pdl=True)
    body(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    g.replay(); torch.cuda.synchronize()
    ts = []
    for it in range(iters):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / layers)
    ts = np.array(ts)
    kv_bytes = float((lay.lens.astype(np.int64)).sum()) * 2 * H * d * 2
    byts = kv_bytes + 2 * lay.batch * Hq * d * 2
    med = np.median(ts)
    print(f"{cfg} tp{tp} {mode} dbg={os.environ.get('BKV_DEBUG', '0')}: B={lay.batch} H={H} Hq={Hq} KV={kv_bytes/1e6:.1f}MB x{layers}  median {med:.1f}us/layer  "
          f"p10 {np.percentile(ts,10):.1f} p90 {np.percentile(ts,90):.1f}  -> {byts/med/1e3:.0f} GB/s "
          f"({byts/med/1e3/6525.9*100:.1f}% of 6526)", flush=True)
    del pools; torch.cuda.empty_cache()

if __name__ == "__main__":
    for spec in sys.argv[1:] or ["opt13b:1", "opt13b:2", "opt30b:4", "llama70b:1", "llama70b:8"]:
        c, t, *m = spec.split(":"); run(c, int(t), mode=m[0] if m else "attn")

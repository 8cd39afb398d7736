"""Quick per-layer timing of decode attention (CUDA events), for development."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case
from synth.workload import shard_heads

def run(cfg, tp=1, layers=8, iters=20):
    sh = CONFIGS[cfg]; case = make_case(cfg, 0); lay = case.layout
    kvh, qh = shard_heads(sh, tp, 0); H = len(kvh); Hq = len(qh); d = sh.head_dim
    dev = "cuda"
    pools = []
    for l in range(layers):
        p = bkv.KVPool(torch.randn(lay.num_blocks, H, sh.block_size, d, device=dev).to(torch.bfloat16),
                       torch.randn(lay.num_blocks, H, sh.block_size, d, device=dev).to(torch.bfloat16))
        pools.append(p)
    bt = torch.from_numpy(lay.block_tables).to(dev); dirs = torch.from_numpy(lay.dirs).to(dev)
    lens = torch.from_numpy(lay.lens).to(dev)
    q = torch.randn(lay.batch, Hq, d, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    for p in pools: bkv.paged_decode_attention(p, bt, dirs, lens, q, out=out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters * layers)]
    k = 0
    for it in range(iters):
        for p in pools:
            ev[k][0].record(); bkv.paged_decode_attention(p, bt, dirs, lens, q, out=out); ev[k][1].record(); k += 1
    torch.cuda.synchronize()
    ts = np.array([a.elapsed_time(b) for a, b in ev]) * 1e3
    kv_bytes = float((lay.lens.astype(np.int64)).sum()) * 2 * H * d * 2
    byts = kv_bytes + 2 * lay.batch * Hq * d * 2
    med = np.median(ts)
    print(f"{cfg} tp{tp}: B={lay.batch} H={H} Hq={Hq} KV={kv_bytes/1e6:.1f}MB  median {med:.1f}us  "
          f"p10 {np.percentile(ts,10):.1f} p90 {np.percentile(ts,90):.1f}  -> {byts/med/1e3:.0f} GB/s  "
          f"({lay.batch/med*1e6/1e6:.2f} M tok/s per layer)", flush=True)

if __name__ == "__main__":
    for spec in sys.argv[1:] or ["opt13b:1", "opt13b:2", "opt30b:4", "llama70b:1", "llama70b:8"]:
        c, t = spec.split(":"); run(c, int(t))

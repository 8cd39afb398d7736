#!/usr/bin/env python
"""BASELINE.json configs[4]: RT:BE ratio and context-length sweep (512-8K, block 16/32) on
the Llama-2-70B shape, per-layer decode attention (fused decode step, CUDA graph over
rotated layers > L2, CUDA events) at the TP1/2/4/8 head shards, through the planned decode
(bkv_decode_plan once, bkv_decode_planned per layer; its large problems take the dynamic
kernel pair).  One JSON line per point: median, p10 and p90 over the replays.

    python scripts/sweep_bench.py [--tp 1 2 4 8] [--L0 512 2048 8192] [--bs 16 32] [--rt 1 0.5 0]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--L0", type=int, nargs="+", default=[512, 1024, 2048, 4096, 8192])
    ap.add_argument("--bs", type=int, nargs="+", default=[16, 32])
    ap.add_argument("--rt", type=float, nargs="+", default=[1.0, 0.5, 0.0])
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    import torch
    import paper_2504_09590_b200 as bkv
    from synth import make_case
    from synth.workload import shard_heads, sweep_shape
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        src = "measured"
    except Exception:
        peak, src = 6650.0, "fallback"
    dev = torch.device("cuda", 0)
    for tp in a.tp:
        for bs in a.bs:
            for L0 in a.L0:
                for rt in a.rt:
                    sh = sweep_shape(L0, bs, rt)
                    lay = make_case(sh, 0).layout
                    kvh, qh = shard_heads(sh, tp, 0)
                    H, Hq, d = len(kvh), len(qh), sh.head_dim
                    kv_bytes = float(lay.lens.astype(np.int64).sum()) * 4 * H * d
                    layers = max(2, min(16, int(math.ceil(600e6 / kv_bytes))))
                    pools = [bkv.KVPool(torch.randn(lay.num_blocks, H, bs, d, device=dev).to(torch.bfloat16),
                                        torch.randn(lay.num_blocks, H, bs, d, device=dev).to(torch.bfloat16))
                             for _ in range(layers)]
                    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
                    bt, dirs, lens = t(lay.block_tables), t(lay.dirs), t(lay.lens.astype(np.int32))
                    q = torch.randn(lay.batch, Hq, d, device=dev).to(torch.bfloat16)
                    kn = torch.randn(lay.batch, H, d, device=dev).to(torch.bfloat16)
                    vn = torch.randn_like(kn)
                    out = torch.empty_like(q)
                    ws = bkv.workspace(lay.batch, Hq, H, d, dev)
                    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pools[0], Hq)

                    def body():
                        for pl in pools:
                            bkv.decode_planned(pl, bt, dirs, lens, plan, q, k_new=kn, v_new=vn, out=out, ws=ws,
                                               pdl=True, kv_early=True)
                    body()
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        body()
                    g.replay()
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(a.iters):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record()
                        g.replay()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e3 / layers)
                    us = float(np.median(ts))
                    nb = lay.nblocks().astype(np.int64)   # bench.py's algorithmic bytes (+ the fused append)
                    alg = kv_bytes + 4.0 * lay.batch * Hq * d + 8.0 * lay.batch * H * d + nb.sum() * 5 + 4 * lay.batch
                    print(json.dumps({"config": "sweep (BASELINE configs[4])", "tp": tp, "block_size": bs, "L0": L0,
                                      "rt_fraction": rt, "batch": lay.batch, "kv_heads": H, "q_heads": Hq,
                                      "mean_ctx": float(lay.lens.mean()), "shared_blocks": int(lay.n_shared),
                                      "us_per_layer": us, "us_p10": float(np.percentile(ts, 10)),
                                      "us_p90": float(np.percentile(ts, 90)),
                                      "plan_blocks_per_warp": plan.header["P"],
                                      "decode_tokens_per_s_per_layer": lay.batch / (us * 1e-6),
                                      "achieved_gbs": alg / (us * 1e-6) / 1e9, "frac": alg / (us * 1e-6) / 1e9 / peak,
                                      "peak_gbs": peak, "peak_source": src}), flush=True)
                    del pools, g
                    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

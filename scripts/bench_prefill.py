#!/usr/bin/env python
"""Measurement of mixed prefill + decode attention on one B200.

    python scripts/bench_prefill.py [--config llama70b] [--tp 1] [--prefill 16] [--steps 20]
                                    [--cost-model gpurun_out/cost_model.csv]

Workload: the config's seeded decode batch (ShareGPT/LMSYS-like
RT lengths, BE prompts U[512,1024]) in which ``--prefill``
BE requests are prefilling their whole prompt (n = L, chunked prefill of a new
request) and every other request decodes one token (n = 1) -- the mixed batch
BROS dispatches per iteration.  One launch of
bkv_paged_prefill_attention per layer, layers rotated so the pools exceed L2,
CUDA graph, CUDA events on the launching stream.

Prints ONE JSON line: achieved TFLOP/s (causal QK^T + PV flops: 4*d per
(query, key) pair per q head) against the bf16 tensor roofline (measured
MEASURED_PEAKS.json bf16_tflops, else the 1.59 PF/s fallback of
B200_PROFILING.md), plus the HBM view (KV bytes of the batch / time).

--cost-model writes per-layer latency samples in SPEC.md's profile CSV
(`phase,l_n,l_a,latency_us`) on the paper's 2^k grid: prefill
samples (l_a = l_n, nothing cached) and decode samples (l_n = batch, l_a = sum
of contexts), and prints the least-squares alpha0/alpha1/beta fit.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["bf16_tflops"]), float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md: 1.59 PFLOP/s bf16, 6.65 TB/s)"


def causal_flops(lens, n, Hq, d):
    """4*d flops per (query, attended key) pair per q head; query i of r sees L-n+i+1 keys."""
    tot = 0
    for L, k in zip(lens.tolist(), n.tolist()):
        # sum_{i<k} (L - k + i + 1) = k*(L-k) + k*(k+1)/2
        tot += k * (L - k) + k * (k + 1) // 2
    return 4.0 * d * Hq * tot


def time_graph(fn, layers, iters, warmup=3):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(iters):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / layers)
    return float(np.median(ts)), ts


def setup(shape, lay, tp, layers, n, seed=0, device="cuda", n_prefill=None):
    import torch
    import paper_2504_09590_b200 as bkv
    from synth import q_rows_torch
    from synth.workload import shard_heads
    kvh, qh = shard_heads(shape, tp, 0)
    H, Hq, d, bs = len(kvh), len(qh), shape.head_dim, shape.block_size
    pools = [bkv.KVPool(torch.randn(lay.num_blocks, H, bs, d, device=device).to(torch.bfloat16),
                        torch.randn(lay.num_blocks, H, bs, d, device=device).to(torch.bfloat16))
             for _ in range(layers)]
    cu = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    q = torch.cat([q_rows_torch(seed, 0, r, int(n[r]), qh, d, shape.num_q_heads, device)
                   for r in range(lay.batch)], 0)
    out = torch.empty_like(q)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
    args = (t(lay.block_tables), t(lay.dirs), t(lay.lens.astype(np.int32)), t(cu))
    max_n = int(n.max())
    if n_prefill is not None:   # P:762-765 dispatch: prefill rows first, then one-row decodes
        rows_p = int(cu[n_prefill])
        max_np = int(n[:n_prefill].max()) if n_prefill else 0
        ws = bkv.workspace(max(1, lay.batch - n_prefill), Hq, H, d, torch.device(device))
        max_len = int(lay.lens.max())

        def fn():
            for p in pools:
                bkv.paged_mixed_attention(p, *args, q, n_prefill, rows_p, max_q_len=max_np,
                                          max_seq_len=max_len, out=out, ws=ws, pdl=True)
        return fn, H, Hq, d

    def fn():
        for p in pools:
            bkv.paged_prefill_attention(p, *args, q, max_q_len=max_n, out=out)
    return fn, H, Hq, d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama70b")
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--prefill", type=int, default=16, help="BE requests prefilling their whole prompt")
    ap.add_argument("--no-decodes", action="store_true", help="only the prefill rows (n = 0 elsewhere)")
    ap.add_argument("--prefill-batch", action="store_true",
                    help="with --no-decodes: the batch holds only the prefill requests (their block tables and "
                         "lengths), as a prefill-only call would pass them; default keeps the whole batch with "
                         "n = 0 for the other requests")
    ap.add_argument("--one-kernel", action="store_true",
                    help="serve the whole mixed batch with the prefill kernel (default: P:762-765 dispatch, "
                         "prefill kernel + split-K decode kernel via bkv_paged_mixed_attention)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cost-model", default=None, help="write phase,l_n,l_a,latency_us samples here")
    a = ap.parse_args()
    import torch
    from synth import CONFIGS, make_case
    from synth.workload import build_layout
    shape = CONFIGS[a.config]
    case = make_case(shape, a.seed)
    lay = case.layout
    rng = np.random.default_rng(a.seed + 1)
    be = np.flatnonzero(lay.is_be)
    pre = rng.choice(be, size=min(a.prefill, be.size), replace=False)
    n = np.zeros(lay.batch, np.int32) if a.no_decodes else np.ones(lay.batch, np.int32)
    n[pre] = lay.lens[pre]
    prefill_tokens = int(n[pre].sum())
    kv_bytes = float(lay.lens.astype(np.int64).sum()) * 4 * shape.head_dim * (shape.num_kv_heads // a.tp)
    layers = max(4, int(math.ceil(500e6 / kv_bytes)))
    dispatch = not a.one_kernel and not a.no_decodes
    if a.no_decodes and a.prefill_batch:   # the prefill requests alone (same pool, same block ids)
        from dataclasses import replace
        lay = replace(lay, lens=lay.lens[pre], is_be=lay.is_be[pre], block_tables=lay.block_tables[pre],
                      dirs=lay.dirs[pre])
        n = n[pre]
        kv_bytes = float(lay.lens.astype(np.int64).sum()) * 4 * shape.head_dim * (shape.num_kv_heads // a.tp)
    if dispatch:   # reorder the batch: prefill requests first (the paper's batch layout)
        from dataclasses import replace
        perm = np.concatenate([pre, np.setdiff1d(np.arange(lay.batch), pre)])
        lay = replace(lay, lens=lay.lens[perm], is_be=lay.is_be[perm], block_tables=lay.block_tables[perm],
                      dirs=lay.dirs[perm])
        n = n[perm]
    fn, H, Hq, d = setup(shape, lay, a.tp, layers, n, a.seed, n_prefill=len(pre) if dispatch else None)
    med, ts = time_graph(fn, layers, a.steps)
    flops = causal_flops(lay.lens.astype(np.int64), n.astype(np.int64), Hq, d)
    tpk, hbm, src = peaks()
    achieved = flops / (med * 1e-6) / 1e12
    line = {
        "metric": "mixed prefill+decode paged attention TFLOP/s (per layer)",
        "value": achieved, "unit": "TFLOP/s", "n_gpus": 1, "steps": a.steps, "higher_is_better": True,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{a.config} TP{a.tp} shard: {H} kv / {Hq} q heads x d{d}, bs{shape.block_size}, "
                               f"batch {lay.batch}: {len(pre)} BE requests prefilling their whole prompt "
                               f"(n = L), {int((n == 1).sum())} decodes (n = 1)",
                   "prefill_tokens": prefill_tokens, "decode_tokens": int((n == 1).sum()),
                   "prefill_batch": bool(a.no_decodes and a.prefill_batch),
                   "layers_rotated": layers, "l2": "pools rotated, > L2", "cuda_graphs": True,
                   "dispatch": ("bkv_paged_mixed_attention: prefill kernel + split-K decode kernel"
                                if dispatch else "bkv_paged_prefill_attention for every row")},
        "us_per_layer": med, "p10_us": float(np.percentile(ts, 10)), "p90_us": float(np.percentile(ts, 90)),
        "roofline": {"bound": "tensor", "kernel": ("bkv::prefill_tc_kernel (tcgen05, TMEM accumulators)"
                                                   if d == 128 and os.environ.get("BKV_PREFILL_MMA_SYNC") != "1"
                                                   else "bkv::prefill_kernel (mma.sync m16n8k16 bf16)")
                     + (" + bkv::decode_kernel" if dispatch else ""),
                     "achieved": achieved, "peak": tpk, "unit": "TFLOP/s", "frac": achieved / tpk,
                     "peak_source": src, "flops_per_launch": flops},
        "hbm_view": {"kv_bytes_per_launch": kv_bytes, "achieved_gbs": kv_bytes / (med * 1e-6) / 1e9,
                     "peak_gbs": hbm},
        "gpu_launches_per_step": layers,
    }
    print(json.dumps(line), flush=True)

    if a.cost_model:
        rows = []
        # prefill samples (one dummy sequence of 2^k tokens; nothing cached: l_a = l_n)
        for ln in (128, 256, 512, 1024, 2048, 4096):
            nreq = 1
            lens = np.full(nreq, ln, np.int64)
            lay2 = build_layout(lens, np.zeros(nreq, bool), shape.block_size, rng, spare_blocks=1)
            fn2, *_ = setup(shape, lay2, a.tp, 4, lens.astype(np.int32), a.seed)
            t2, _ = time_graph(fn2, 4, 10)
            rows.append(("Prefill", int(lens.sum()), int(lens.sum()), t2))
        # decode samples: l_n = batch (one new token each), l_a = attended tokens
        for B in (16, 64, 256):
            for L in (256, 1024, 4096):
                lens = np.full(B, L, np.int64)
                lay2 = build_layout(lens, np.arange(B) % 2 == 1, shape.block_size, rng, spare_blocks=1)
                fn2, *_ = setup(shape, lay2, a.tp, 4, np.ones(B, np.int32), a.seed)
                t2, _ = time_graph(fn2, 4, 10)
                rows.append(("Decode", B, int(lens.sum()), t2))
        os.makedirs(os.path.dirname(os.path.abspath(a.cost_model)), exist_ok=True)
        with open(a.cost_model, "w") as f:
            f.write("phase,l_n,l_a,latency_us\n")
            for ph, ln, la, t in rows:
                f.write(f"{ph},{ln},{la},{t:.3f}\n")
        fit = {}
        for ph in ("Prefill", "Decode"):
            X = np.array([[r[1], r[1] * r[2], 1.0] for r in rows if r[0] == ph], float)
            y = np.array([r[3] for r in rows if r[0] == ph], float)
            c, *_ = np.linalg.lstsq(X, y, rcond=None)
            c = np.maximum(c, 0.0)
            fit[ph.lower()] = {"alpha0": c[0], "alpha1": c[1], "beta": c[2]}
        print(json.dumps({"cost_model_fit_per_layer_attention": fit, "samples": len(rows)}), flush=True)


if __name__ == "__main__":
    main()

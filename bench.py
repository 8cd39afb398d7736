#!/usr/bin/env python
"""Benchmark of the BROS bidirectional paged decode-attention hot path on B200.

One STEP = one decode iteration of the attention path over ALL layers of the
model shape: per layer, kv_append of the batch's new tokens
and paged decode attention over the bidirectional block map (a3-a5); at N > 1
GPUs each rank owns a head shard (tensor parallel by kv head) and the
head-major outputs of every layer are reassembled with ONE NCCL all-gather per
step (a6; ``--gather layer``: one per layer, ``--reassembly p2p``: peer stores).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config opt13b] [--impl reference]

Prints ONE JSON line (rank 0).  ``value`` = decode tokens/s of the whole job
(batch tokens per step / device step time, max over ranks).  Per-layer KV data
is far larger than L2 and every step sweeps every layer's pool once, so no
explicit L2 flush is needed ("inputs larger than L2").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn tokens/s and achieved HBM GB/s vs B200 peak at 1/2/4/8 GPUs"
WORKLOADS = {
    "opt13b": "OPT-13B shape: 40 heads x d128, bs16, ShareGPT-like lengths, mixed RT/BE batch 64 (1:1, shared tails), 40 layers",
    "opt30b": "OPT-30B shape: 56 heads x d128, bs16, LMSYS-like lengths, mixed RT/BE batch 128, 48 layers",
    "llama70b": "Llama-2-70B shape: 64 Q / 8 KV heads (GQA 8) x d128, bs16, ShareGPT-like lengths, batch 256, 80 layers",
    "tiny": "tiny: 4 heads x d64, bs16, 8 requests (4 RT + 4 BE) sharing blocks, ctx <= 256, 1 layer",
}


# ------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """dram read+write bytes per attention launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def algorithmic_bytes(lay, H, Hq, d, bs):
    """Bytes one attention launch must move: KV of every resident
    token for the local kv heads, q and out rows, block-table + direction entries
    and seq_lens."""
    L = lay.lens.astype(np.int64)
    nb = lay.nblocks().astype(np.int64)        # entries: ceil(L/bs), or num_entries of a general map
    kv = float(L.sum()) * 2 * H * d * 2
    qo = 2.0 * lay.batch * Hq * d * 2
    per_entry = 4 + 1 + (1 if lay.general else 0)   # block id, direction (+ fill count)
    meta = float(nb.sum()) * per_entry + (8.0 if lay.general else 4.0) * lay.batch
    return kv + qo + meta, kv


def append_bytes(B, H, d):
    return 8.0 * B * H * d   # read k_new, v_new + write the two rows: 4 x B*H*d bf16 values


# --------------------------------------------------------- reference (oracle) arm
def host_cores(oracle):
    """Let the oracle use every core this process may run on."""
    try:
        n = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        n = os.cpu_count() or 1
    oracle.set_num_threads(max(1, n))


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from synth import CONFIGS, make_case
    sh = CONFIGS[args.config]
    case = make_case(args.config, args.seed)
    lay = case.layout
    H, Hq, d, bs, B = sh.num_kv_heads, sh.num_q_heads, sh.head_dim, sh.block_size, lay.batch
    rng = np.random.default_rng(1)
    # bounded sample: one layer of the workload, all requests, first `heads` kv heads
    heads = max(1, min(H, args.ref_heads))
    g = sh.group
    K = (rng.standard_normal((lay.num_blocks, heads, bs, d), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    V = (rng.standard_normal((lay.num_blocks, heads, bs, d), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    q = (rng.standard_normal((B, heads * g, d), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    host_cores(oracle)   # rank 0 runs alone: all host cores (torchrun sets OMP_NUM_THREADS=1)
    cores = oracle.num_threads()
    W = args.warmup if args.warmup_ref is None else args.warmup_ref
    times = []
    for i in range(W + args.steps):
        t0 = time.perf_counter()
        oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 1.0 / math.sqrt(d))
        dt = time.perf_counter() - t0
        if i >= W:
            times.append(dt)
    t_layer_full = statistics.median(times) * (H / heads)        # scale the head sample to all heads
    t_step = t_layer_full * sh.n_layers
    value = B / t_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": W, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "name": args.config,
                   "global_batch": B, "n_layers": sh.n_layers, "tp": 1},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"one layer, all {B} requests, {heads}/{H} kv heads "
                                   f"({heads * g} q heads) of {args.config}; time scaled by "
                                   f"{H}/{heads} heads x {sh.n_layers} layers; median of {len(times)}"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, lay, sh):
    """The oracle as it stands, timed on the host cores on a bounded sample."""
    import oracle
    H, Hq, d, bs, B = sh.num_kv_heads, sh.num_q_heads, sh.head_dim, sh.block_size, lay.batch
    heads = max(1, min(H, args.ref_heads))
    g = sh.group
    host_cores(oracle)
    rng = np.random.default_rng(2)
    K = (rng.standard_normal((lay.num_blocks, heads, bs, d), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    V = (rng.standard_normal((lay.num_blocks, heads, bs, d), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    q = (rng.standard_normal((B, heads * g, d), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    ts = []
    t_end = time.perf_counter() + args.cpu_seconds
    while len(ts) < 3 and (not ts or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 1.0 / math.sqrt(d))
        ts.append(time.perf_counter() - t0)
    t_step = statistics.median(ts) * (H / heads) * sh.n_layers
    return {"value": B / t_step, "unit": "tokens/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"one layer, all {B} requests, {heads}/{H} kv heads of {args.config}, "
                      f"median of {len(ts)} runs, scaled x{H}/{heads} heads x {sh.n_layers} layers"}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_09590_b200 as bkv
    from synth import CONFIGS, make_case
    from paper_2504_09590_b200.tp import HeadShard, PeerReassembly, gather_heads

    ws, rank, local = dist_env()
    # dev-only: BKV_DIST_BACKEND=gloo runs several ranks on one GPU (smoke test of the N>1 path)
    backend = os.environ.get("BKV_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
        if ws > 1 and args.reassembly == "nccl":
            args.graphs = False      # the gloo all-gather goes through host memory: not capturable
    if ws > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    sh = CONFIGS[args.config]
    tp = ws
    if sh.num_kv_heads % tp:
        raise SystemExit(f"{args.config}: {sh.num_kv_heads} kv heads do not shard over {tp} GPUs")
    case = make_case(args.config, args.seed, general=args.general_map)
    lay = case.layout
    shard = HeadShard(sh.num_q_heads, sh.num_kv_heads, tp, rank)
    kv_heads, q_heads = list(shard.kv_heads), list(shard.q_heads)
    H, Hq, d, bs, B = len(kv_heads), len(q_heads), sh.head_dim, sh.block_size, lay.batch
    n_layers = args.layers or sh.n_layers
    stream = torch.cuda.current_stream(dev)

    # ---- resident state: one KV pool per layer (random bf16 contents), block map
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    pools = []
    for _ in range(n_layers):
        k = torch.empty((lay.num_blocks, H, bs, d), dtype=torch.bfloat16, device=dev)
        v = torch.empty_like(k)
        k.normal_(generator=gen)
        v.normal_(generator=gen)
        pools.append(bkv.KVPool(k, v))
    # ---- per-step inputs (host-pinned originals for the e2e leg)
    before_h = torch.from_numpy((lay.lens - 1).astype(np.int32))
    cu_h = torch.arange(B + 1, dtype=torch.int32)
    meta_h = {
        "bt": torch.from_numpy(lay.block_tables).pin_memory(),
        "dirs": torch.from_numpy(lay.dirs).pin_memory(),
        "lens": torch.from_numpy(lay.lens.astype(np.int32)).pin_memory(),
        "before": before_h.pin_memory(),
        "cu": cu_h.pin_memory(),
    }
    if args.general_map:   # per-entry fill counts travel with the map
        meta_h["fills"] = torch.from_numpy(lay.fills).pin_memory()
        meta_h["nent"] = torch.from_numpy(lay.num_entries).pin_memory()
    g_cpu = torch.Generator().manual_seed(99)
    q_h = torch.randn((n_layers, B, Hq, d), generator=g_cpu).to(torch.bfloat16).pin_memory()
    kn_h = torch.randn((n_layers, B, H, d), generator=g_cpu).to(torch.bfloat16).pin_memory()
    vn_h = torch.randn((n_layers, B, H, d), generator=g_cpu).to(torch.bfloat16).pin_memory()
    meta_d = {k: v.to(dev) for k, v in meta_h.items()}
    q_d, kn_d, vn_d = q_h.to(dev), kn_h.to(dev), vn_h.to(dev)
    out_loc = torch.empty((n_layers, Hq, B, d), dtype=torch.bfloat16, device=dev)   # head-major
    # reassembled outputs: per-layer gather -> [layer][global head][B][d]; one gather per step
    # (default) -> rank-major [rank][layer][local head][B][d] (global head = rank * Hq + local)
    glob_shape = (n_layers, Hq * tp, B, d) if args.gather == "layer" else (tp, n_layers, Hq, B, d)
    out_glob = torch.empty(glob_shape, dtype=torch.bfloat16, device=dev) if tp > 1 else None
    p2p = None
    if tp > 1 and args.reassembly == "p2p":   # f2: fused NVLink reassembly instead of the all-gather
        p2p = PeerReassembly(shard, n_layers, B, d, dev)
        out_glob = p2p.glob
    out_h = torch.empty(tuple(out_glob.shape) if out_glob is not None else (n_layers, Hq, B, d),
                        dtype=torch.bfloat16).pin_memory()
    wsb = bkv.workspace(B, Hq, H, d, dev)
    max_len = int(lay.lens.max())
    scale = 1.0 / math.sqrt(d)

    def step(md, qd, knd, vnd, attn_only=False, ol=None, og=None):
        """One decode step over all layers (append + attention [+ all-gather])."""
        ol = out_loc if ol is None else ol
        og = out_glob if og is None else og
        launches = 0
        gm = dict(fills=md["fills"], num_entries=md["nent"]) if args.general_map else {}
        for l in range(n_layers):
            if p2p is not None:   # f2: fused step + stores into every peer's output, then signal
                bkv.decode_multi_out(pools[l], md["bt"], md["dirs"], md["lens"], qd[l],
                                     p2p.local_out(l).permute(1, 0, 2), p2p.peer_outs(l),
                                     k_new=knd[l], v_new=vnd[l], softmax_scale=scale,
                                     max_seq_len=max_len, ws=wsb, pdl=args.pdl, **gm)
                launches += 2
                if not attn_only:
                    p2p.barrier()
                    launches += 1
                continue
            o = ol[l].permute(1, 0, 2)                                        # [B][Hq][d] view
            if args.fused:   # f2: append fused into the attention kernel (bkv_decode_step)
                bkv.decode_step(pools[l], md["bt"], md["dirs"], md["lens"], knd[l], vnd[l], qd[l],
                                scale, out=o, max_seq_len=max_len, ws=wsb, pdl=args.pdl, **gm)
            else:
                if not attn_only:
                    bkv.kv_append(pools[l], md["bt"], md["dirs"], md["before"], md["cu"], knd[l],
                                  vnd[l], total_new_tokens=B, **gm)
                    launches += 1
                bkv.paged_decode_attention(pools[l], md["bt"], md["dirs"], md["lens"], qd[l], scale,
                                           out=o, max_seq_len=max_len, ws=wsb, pdl=args.pdl, **gm)
            launches += 2                                                     # decode + merge kernels
            if tp > 1 and not attn_only and args.gather == "layer":
                gather_heads(ol[l], og[l])
        if tp > 1 and not attn_only and p2p is None and args.gather == "step":
            # a6: head-sharded TP needs no per-layer reassembly (each rank's o_proj shard
            # consumes its own heads); the step's per-request outputs of every layer are
            # reassembled by ONE all-gather
            gather_heads(ol.view(n_layers * Hq, B, d), og.view(tp * n_layers * Hq, B, d))
        return launches

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- eager warm-up, then capture the step (and an attention-only step) in CUDA graphs
    for _ in range(args.warmup):
        launches_per_step = step(meta_d, q_d, kn_d, vn_d)
    barrier()
    g_step, g_attn = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    if args.graphs:
        try:
            with torch.cuda.graph(g_step):
                step(meta_d, q_d, kn_d, vn_d)
            with torch.cuda.graph(g_attn):
                step(meta_d, q_d, kn_d, vn_d, attn_only=True)
        except Exception as e:   # e.g. a collective that cannot be captured: time the eager launches
            print(f"bench: CUDA graph capture failed ({type(e).__name__}: {e}); running eagerly",
                  file=sys.stderr, flush=True)
            torch.cuda.synchronize(dev)
            args.graphs = False
    if args.graphs:
        run_step, run_attn = g_step.replay, g_attn.replay
    else:
        run_step = lambda: step(meta_d, q_d, kn_d, vn_d)
        run_attn = lambda: step(meta_d, q_d, kn_d, vn_d, attn_only=True)
    for _ in range(args.warmup):
        run_step()
    barrier()

    def timed(fn, n):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    # ---- device-resident timed region (W warm-up steps done above)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)                          # let nvidia-smi attach before the timed region
    ms_total = timed(run_step, args.steps)
    ms_step = ms_total / args.steps
    launches = launches_per_step * args.steps
    # ---- the dominant kernel alone: same pools, attention launches only, same stream
    for _ in range(2):
        run_attn()
    att_avg_us = timed(run_attn, args.steps) * 1e3 / (args.steps * n_layers)

    # ---- end to end: pinned host inputs -> device, step, device -> host outputs
    src_out = out_glob if tp > 1 else out_loc

    def e2e_step():
        for k, v in meta_h.items():
            meta_d[k].copy_(v, non_blocking=True)
        q_d.copy_(q_h, non_blocking=True)
        kn_d.copy_(kn_h, non_blocking=True)
        vn_d.copy_(vn_h, non_blocking=True)
        run_step()
        out_h.copy_(src_out, non_blocking=True)

    pipelined = args.graphs and p2p is None and args.e2e_pipeline
    if pipelined:
        # Serving pipeline: two input/output buffer sets, one captured graph per set; one
        # copy stream moves step i+1's inputs host -> device while step i computes, another
        # step i's outputs device -> host while step i+1 computes (both copy engines busy).  Every step still
        # moves all of its inputs and outputs through PCIe inside the timed region.
        meta_d2 = {k: torch.empty_like(v) for k, v in meta_d.items()}
        q_d2, kn_d2, vn_d2 = torch.empty_like(q_d), torch.empty_like(kn_d), torch.empty_like(vn_d)
        out_loc2 = torch.empty_like(out_loc)
        out_glob2 = torch.empty_like(out_glob) if out_glob is not None else None
        for k in meta_d:
            meta_d2[k].copy_(meta_d[k])
        q_d2.copy_(q_d), kn_d2.copy_(kn_d), vn_d2.copy_(vn_d)
        step(meta_d2, q_d2, kn_d2, vn_d2, ol=out_loc2, og=out_glob2)   # eager warm-up of set 2
        torch.cuda.synchronize(dev)
        g_step2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step2):
            step(meta_d2, q_d2, kn_d2, vn_d2, ol=out_loc2, og=out_glob2)
        sets = [(meta_d, q_d, kn_d, vn_d, g_step, src_out),
                (meta_d2, q_d2, kn_d2, vn_d2, g_step2, out_glob2 if tp > 1 else out_loc2)]
        up = torch.cuda.Stream(dev)     # host -> device (one copy engine) ...
        down = torch.cuda.Stream(dev)   # ... and device -> host (the other), concurrently
        ev_h2d = [torch.cuda.Event(), torch.cuda.Event()]
        ev_comp = [torch.cuda.Event(), torch.cuda.Event()]
        ev_d2h = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(si):
            md, qd, knd, vnd, _, _ = sets[si]
            with torch.cuda.stream(up):
                for k, v in meta_h.items():
                    md[k].copy_(v, non_blocking=True)
                qd.copy_(q_h, non_blocking=True)
                knd.copy_(kn_h, non_blocking=True)
                vnd.copy_(vn_h, non_blocking=True)
                ev_h2d[si].record(up)

        def run_pipeline(n):
            up.wait_stream(stream)
            down.wait_stream(stream)
            h2d(0)
            for i in range(n):
                si = i % 2
                stream.wait_event(ev_h2d[si])
                if i >= 2:                         # step i-2's outputs (same set) are on the host
                    stream.wait_event(ev_d2h[si])
                sets[si][4].replay()
                ev_comp[si].record(stream)
                if i + 1 < n:                      # inputs of step i+1 (its set was last read by step i-1)
                    sj = 1 - si
                    if i >= 1:
                        up.wait_event(ev_comp[sj])
                    h2d(sj)
                with torch.cuda.stream(down):      # outputs of step i, overlapping step i+1
                    down.wait_event(ev_comp[si])
                    out_h.copy_(sets[si][5], non_blocking=True)
                    ev_d2h[si].record(down)
            stream.wait_stream(up)
            stream.wait_stream(down)

        def timed_pipeline(n):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            run_pipeline(n)
            e1.record(stream)
            barrier()
            return max_over_ranks(e0.elapsed_time(e1))

        run_pipeline(2)
        ms_e2e = timed_pipeline(args.steps) / args.steps
    else:
        for _ in range(2):
            e2e_step()
        ms_e2e = timed(e2e_step, args.steps) / args.steps
    if p2p is not None:
        p2p.check()
    clk = clocks.stop()                      # clocks sampled over all three timed regions
    h2d = sum(v.numel() * v.element_size() for v in meta_h.values()) + \
        (q_h.numel() + kn_h.numel() + vn_h.numel()) * 2
    d2h = out_h.numel() * 2

    if rank != 0:
        dist.destroy_process_group()
        return
    alg_bytes, kv_bytes = algorithmic_bytes(lay, H, Hq, d, bs)
    if args.fused:   # the fused kernel also reads the new rows and writes them into the pool
        alg_bytes += append_bytes(B, H, d)
    peak, peak_src = load_peaks()
    achieved = alg_bytes / (att_avg_us * 1e-6) / 1e9
    tok_s = B / (ms_step * 1e-3)
    cpu = cpu_baseline(args, lay, sh) if (ws == 1 and not args.no_cpu) else None
    line = {
        "metric": METRIC,
        "value": tok_s,
        "unit": "tokens/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": {
            "workload": WORKLOADS.get(args.config, args.config), "name": args.config,
            "global_batch": B, "n_layers": n_layers, "parallelism": f"tp{tp} (kv-head sharded)",
            "kv_heads_per_gpu": H, "q_heads_per_gpu": Hq, "head_dim": d, "block_size": bs,
            "mean_ctx": float(lay.lens.mean()), "max_ctx": int(lay.lens.max()),
            "shared_blocks": int(lay.n_shared),
            "block_map": "general (per-entry fills, f3)" if args.general_map else "dense",
            "l2": f"inputs larger than L2: each step reads {n_layers} layers x {kv_bytes / 1e6:.0f} MB of KV per GPU",
            "per_layer_us": ms_step * 1e3 / n_layers,
            "attn_us_per_layer": att_avg_us,
            "attn_share_of_step": att_avg_us * n_layers / (ms_step * 1e3),
            "cuda_graphs": bool(args.graphs),
            "fused_append": bool(args.fused),
            "reassembly": ("p2p stores + peer barrier (bkv_decode_multi_out)" if p2p is not None
                           else f"nccl all_gather_into_tensor, one per {args.gather}" if tp > 1
                           else "none (1 GPU)"),
            "attn_layer_tokens_per_s": B / (att_avg_us * 1e-6),
            "seed": args.seed,
        },
        "roofline": {
            "bound": "hbm", "kernel": "bkv::decode_kernel" + (" (fused append)" if args.fused else ""), "achieved": achieved, "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
            "algorithmic_bytes_per_launch": alg_bytes,
            "traffic": ncu_traffic(f"{args.config}_tp{tp}"),
        },
        "cpu_baseline": cpu,
        "e2e": {"value": B / (ms_e2e * 1e-3), "unit": "tokens/s", "ms_per_step": ms_e2e,
                "pipeline": ("two copy streams overlap step i+1 H2D and step i D2H with compute (2 buffer sets)"
                             if pipelined else "serial H2D, step, D2H on one stream"),
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="opt13b", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--layers", type=int, default=0, help="override the model's layer count")
    ap.add_argument("--ref-heads", type=int, default=4, help="kv heads in the oracle's bounded sample")
    ap.add_argument("--warmup-ref", type=int, default=None, help="reference-arm warm-ups (default: --warmup)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pdl", dest="pdl", action="store_false",
                    help="launch attention without programmatic dependent launch")
    ap.add_argument("--no-e2e-pipeline", dest="e2e_pipeline", action="store_false",
                    help="e2e leg: serial H2D/step/D2H instead of the double-buffered copy-stream pipeline")
    ap.add_argument("--general-map", action="store_true",
                    help="FindBlock-style general block map (partly filled entries, SURVEY §8(f) f3)")
    ap.add_argument("--gather", default="step", choices=["step", "layer"],
                    help="N>1, nccl reassembly: one all-gather per step of every layer's outputs (default) "
                         "or one per layer")
    ap.add_argument("--reassembly", default="nccl", choices=["nccl", "p2p"],
                    help="N>1: NCCL all-gather (default) or fused NVLink stores (symmetric memory)")
    ap.add_argument("--no-fused", dest="fused", action="store_false",
                    help="separate kv_append + attention launches instead of bkv_decode_step")
    ap.add_argument("--no-graphs", dest="graphs", action="store_false",
                    help="launch eagerly instead of replaying CUDA graphs")
    args = ap.parse_args()
    ws, _, _ = dist_env()
    if args.gpus != ws and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {ws}")
    if args.gpus > 1 and ws == 1:
        raise SystemExit("N > 1 must be launched with torch.distributed.run (one process per GPU)")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

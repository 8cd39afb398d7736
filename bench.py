#!/usr/bin/env python
"""Benchmark of the BROS bidirectional paged decode-attention hot path on B200.

One STEP = one decode iteration of the attention path over ALL layers of the
model shape: per layer, this step's new K/V rows are appended into their
bidirectional slots and every request attends over its context (SURVEY §8(a)
a1-a5), fused in one planned-decode call (bkv_decode_planned: the decode kernel
with the append fused in, plus the light cross-CTA merge kernel); the split plan
is built on the host once per step (bkv_decode_plan) and shared by all layers.
At N > 1 GPUs each rank owns a head shard (tensor parallel by kv head)
and the head-major outputs of every layer are reassembled with ONE NCCL
all-gather per step (a6; ``--gather layer``: one per layer; ``--reassembly
p2p``: stores into the peers' outputs over NVLink + a peer barrier, f2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config opt13b] [--impl reference]

Prints ONE JSON line (rank 0).  ``value`` = decode tokens/s of the whole job
(batch tokens per step / device step time, max over ranks).  Per-layer KV data
is far larger than L2 and every step sweeps every layer's pool once ("inputs
larger than L2").  At N = 1 the line also carries ``shards``: the per-layer
time of every head shard the paper runs (Llama-2-70B TP1/2/4/8, OPT-13B
TP2/4/8, OPT-30B TP4) on this GPU, median / p10 / p90 over 60 graph replays.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
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
# the head shards of the paper's deployments and their neighbours, measured at N = 1
SHARDS = [("llama70b", 1), ("llama70b", 2), ("llama70b", 4), ("llama70b", 8),
          ("opt13b", 2), ("opt13b", 4), ("opt13b", 8), ("opt30b", 4)]
L2_BYTES = 126 * 2 ** 20
PLANNED_DYNAMIC_P = 128   # bkv_decode_planned's default switch to the dynamic schedule (include/bkv.h)


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
    """DRAM read+write bytes per layer launch pair from this round's committed ncu capture
    of the same kernels and shard (profiles/r02/ncu_traffic.json); not measured in this run."""
    p = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def pct(xs, q):
    return float(np.percentile(np.asarray(xs, dtype=np.float64), q))


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
    """Bytes one layer's attention must move: KV of every resident token
    for the local kv heads, q and out rows, block-table + direction entries and seq_lens."""
    L = lay.lens.astype(np.int64)
    nb = lay.nblocks().astype(np.int64)        # entries: ceil(L/bs), or num_entries of a general map
    kv = float(L.sum()) * 2 * H * d * 2
    qo = 2.0 * lay.batch * Hq * d * 2
    per_entry = 4 + 1 + (1 if lay.general else 0)   # block id, direction (+ fill count)
    meta = float(nb.sum()) * per_entry + (8.0 if lay.general else 4.0) * lay.batch
    return kv + qo + meta, kv


def append_bytes(B, H, d):
    return 8.0 * B * H * d   # read k_new, v_new + write the two rows: 4 x B*H*d bf16 values


def workload_config(args, ws, sh, lay):
    """The config object both arms print (same keys, so the driver can compare them)."""
    return {"workload": WORKLOADS.get(args.config, args.config), "name": args.config,
            "global_batch": int(lay.batch), "n_layers": int(args.layers or sh.n_layers),
            "parallelism": f"tp{ws} (kv-head sharded)", "head_dim": sh.head_dim,
            "block_size": sh.block_size, "num_q_heads": sh.num_q_heads, "num_kv_heads": sh.num_kv_heads,
            "block_map": "general (per-entry fills, f3)" if args.general_map else "dense",
            "seed": args.seed,
            "l2": "inputs larger than L2: every step reads every layer's KV pool once"}


# --------------------------------------------------------- oracle timing (CPU)
def oracle_layer(sh, lay, seed=2):
    """One full layer of the workload (all heads, all requests) as host arrays for the oracle."""
    H, d, bs, B = sh.num_kv_heads, sh.head_dim, sh.block_size, lay.batch
    rng = np.random.default_rng(seed)
    bf = lambda shape: (rng.standard_normal(shape, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    return bf((lay.num_blocks, H, bs, d)), bf((lay.num_blocks, H, bs, d)), bf((B, sh.num_q_heads, d))


def time_oracle_layer(oracle, K, V, lay, q, d, threads, reps):
    oracle.set_num_threads(threads)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 1.0 / math.sqrt(d))
        ts.append(time.perf_counter() - t0)
    return ts


def run_reference(args):
    """The reference arm of the tier framing: the CPU oracle as it stands, on the host cores.
    One step = one full layer of the workload (every head, every request); value = the
    batch's tokens / (measured per-layer time x the model's layers)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from synth import CONFIGS, make_case
    sh = CONFIGS[args.config]
    lay = make_case(args.config, args.seed).layout
    n_layers = args.layers or sh.n_layers
    K, V, q = oracle_layer(sh, lay)
    cores = host_cores()   # rank 0 runs alone: all host cores (torchrun sets OMP_NUM_THREADS=1)
    times = time_oracle_layer(oracle, K, V, lay, q, sh.head_dim, cores, args.warmup + args.steps)[args.warmup:]
    one = time_oracle_layer(oracle, K, V, lay, q, sh.head_dim, 1, 1)[0]
    t_layer = statistics.median(times)
    value = lay.batch / (t_layer * n_layers)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(times)) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args, ws, sh, lay),
        "step_definition": f"one full layer of the workload (all {sh.num_q_heads} q heads, all {lay.batch} "
                           f"requests) per step; value = batch / (median layer time x {n_layers} layers)",
        "step_ms": {"median": t_layer * 1e3, "p10": pct(times, 10) * 1e3, "p90": pct(times, 90) * 1e3},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"one full layer ({sh.num_q_heads} q heads x {lay.batch} requests) of "
                                   f"{args.config} per step, fp64 C oracle with OpenMP",
                         "layer_ms_all_cores": t_layer * 1e3, "layer_ms_1_thread": one * 1e3,
                         "value_1_thread": lay.batch / (one * n_layers)},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, lay, sh, n_layers):
    """The oracle as it stands, timed on the host cores on a bounded sample: one full layer."""
    import oracle
    K, V, q = oracle_layer(sh, lay)
    cores = host_cores()
    ts = time_oracle_layer(oracle, K, V, lay, q, sh.head_dim, cores, 3)
    one = time_oracle_layer(oracle, K, V, lay, q, sh.head_dim, 1, 1)[0]
    t = statistics.median(ts)
    return {"value": lay.batch / (t * n_layers), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"one full layer ({sh.num_q_heads} q heads x {lay.batch} requests) of {args.config}, "
                      f"median of 3 at {cores} threads, scaled x {n_layers} layers",
            "layer_ms_all_cores": t * 1e3, "layer_ms_1_thread": one * 1e3,
            "value_1_thread": lay.batch / (one * n_layers)}


# ------------------------------------------------------------------ shards
def measure_shards(dev, peak, seed, replays=60, warm=10):
    """Per-layer time of every head shard of the paper's deployments on this GPU: the
    planned fused decode step per layer in a CUDA graph over >= 4x L2 of rotated layers."""
    import torch
    import paper_2504_09590_b200 as bkv
    from synth import CONFIGS, make_case
    from synth.workload import shard_heads
    res = []
    for cfg, tp in SHARDS:
        sh = CONFIGS[cfg]
        lay = make_case(cfg, seed).layout
        kvh, qh = shard_heads(sh, tp, 0)
        H, Hq, d, bs, B = len(kvh), len(qh), sh.head_dim, sh.block_size, lay.batch
        alg, kv = algorithmic_bytes(lay, H, Hq, d, bs)
        alg += append_bytes(B, H, d)
        layers = max(8, math.ceil(4 * L2_BYTES / kv))
        gen = torch.Generator(device=dev).manual_seed(7)
        pools = []
        for _ in range(layers):
            k = torch.empty((lay.num_blocks, H, bs, d), dtype=torch.bfloat16, device=dev).normal_(generator=gen)
            pools.append(bkv.KVPool(k, torch.empty_like(k).normal_(generator=gen)))
        bt = torch.from_numpy(lay.block_tables).to(dev)
        dirs = torch.from_numpy(lay.dirs).to(dev)
        lens = torch.from_numpy(lay.lens.astype(np.int32)).to(dev)
        q = torch.randn((layers, B, Hq, d), device=dev).to(torch.bfloat16)
        kn = torch.randn((layers, B, H, d), device=dev).to(torch.bfloat16)
        vn = torch.randn((layers, B, H, d), device=dev).to(torch.bfloat16)
        out = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=dev)
        ws = bkv.workspace(B, Hq, H, d, dev)
        plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pools[0], Hq)

        def body():
            for l in range(layers):
                bkv.decode_planned(pools[l], bt, dirs, lens, plan, q[l], k_new=kn[l], v_new=vn[l], out=out,
                                   ws=ws, pdl=True, kv_early=True)
        body()
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        for _ in range(warm):
            g.replay()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(replays + 1)]
        torch.cuda.synchronize(dev)
        evs[0].record()
        for i in range(replays):
            g.replay()
            evs[i + 1].record()
        torch.cuda.synchronize(dev)
        us = [evs[i].elapsed_time(evs[i + 1]) * 1e3 / layers for i in range(replays)]
        med = statistics.median(us)
        res.append({"shard": f"{cfg} tp{tp}", "kv_heads": H, "q_heads": Hq, "batch": B,
                    "kv_mb_per_layer": kv / 1e6, "alg_mb_per_layer": alg / 1e6, "layers_rotated": layers,
                    "us_per_layer": {"median": med, "p10": pct(us, 10), "p90": pct(us, 90)},
                    "gbs": alg / (med * 1e-6) / 1e9, "frac": alg / (med * 1e-6) / 1e9 / peak,
                    "traffic": ncu_traffic(f"{cfg}_tp{tp}")})
        del pools, g, q, kn, vn
        torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ our arm
def run_ours(args):
    ws, rank, local = dist_env()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # NCCL's init log (rank count, NVLS/NVLink) on stderr
    import torch
    import torch.distributed as dist

    import paper_2504_09590_b200 as bkv
    from synth import CONFIGS, make_case
    from paper_2504_09590_b200.tp import HeadShard, MulticastReassembly, PeerReassembly, gather_heads

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
    bt_stride = lay.block_tables.shape[1]

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
    # ---- per-step inputs (host-pinned originals for the e2e leg), incl. the step's split plan
    nent_h = lay.num_entries if args.general_map else None

    def host_plan():   # the host scheduler's plan of the step: lengths + block map -> flattened work list
        return bkv.decode_plan_host(lay.lens, lay.block_tables, lay.dirs, H, Hq, d, bs,
                                    fills=lay.fills if args.general_map else None, num_entries=nent_h)

    plan_np = host_plan()
    meta_h = {
        "bt": torch.from_numpy(lay.block_tables).pin_memory(),
        "dirs": torch.from_numpy(lay.dirs).pin_memory(),
        "lens": torch.from_numpy(lay.lens.astype(np.int32)).pin_memory(),
        "plan": torch.from_numpy(plan_np.view(np.uint8).copy()).pin_memory(),
    }
    if args.general_map:   # per-entry fill counts travel with the map
        meta_h["fills"] = torch.from_numpy(lay.fills).pin_memory()
        meta_h["nent"] = torch.from_numpy(lay.num_entries).pin_memory()
    g_cpu = torch.Generator().manual_seed(99)
    q_h = torch.randn((n_layers, B, Hq, d), generator=g_cpu).to(torch.bfloat16).pin_memory()
    kn_h = torch.randn((n_layers, B, H, d), generator=g_cpu).to(torch.bfloat16).pin_memory()
    vn_h = torch.randn((n_layers, B, H, d), generator=g_cpu).to(torch.bfloat16).pin_memory()

    def dev_meta():
        md = {k: v.to(dev) for k, v in meta_h.items()}
        md["plan_obj"] = bkv.DecodePlan(plan_np, md["plan"], md["plan"].numel())
        return md

    meta_d = dev_meta()
    q_d, kn_d, vn_d = q_h.to(dev), kn_h.to(dev), vn_h.to(dev)
    out_loc = torch.empty((n_layers, Hq, B, d), dtype=torch.bfloat16, device=dev)   # head-major
    # reassembled outputs: per-layer gather -> [layer][global head][B][d]; one gather per step
    # (default) -> rank-major [rank][layer][local head][B][d] (global head = rank * Hq + local)
    glob_shape = (n_layers, Hq * tp, B, d) if args.gather == "layer" else (tp, n_layers, Hq, B, d)
    fused = tp > 1 and args.reassembly in ("p2p", "nvls")
    n_sets = 3 if fused else 2   # e2e buffer sets (fused reassembly: triple)
    p2ps = None
    if fused:   # f2: fused NVLink reassembly (peer stores, or NVLS multicast stores) instead of the all-gather
        R = MulticastReassembly if args.reassembly == "nvls" else PeerReassembly
        p2ps = [R(shard, n_layers, B, d, dev) for _ in range(n_sets)]
        out_glob = p2ps[0].glob
    else:
        out_glob = torch.empty(glob_shape, dtype=torch.bfloat16, device=dev) if tp > 1 else None
    out_h = torch.empty(tuple(out_glob.shape) if out_glob is not None else (n_layers, Hq, B, d),
                        dtype=torch.bfloat16).pin_memory()
    wsb = bkv.workspace(B, Hq, H, d, dev)
    scale = 1.0 / math.sqrt(d)

    def step(md, qd, knd, vnd, ol, og, p2p=None, attn_only=False, gather_only=False):
        """One decode step over all layers (planned fused append + attention [+ reassembly])."""
        launches = 0
        gm = dict(fills=md["fills"], num_entries=md["nent"]) if args.general_map else {}
        if not gather_only:
            for l in range(n_layers):
                if p2p is not None:   # f2: the layer's rows are also stored into every peer's output
                    bkv.decode_planned(pools[l], md["bt"], md["dirs"], md["lens"], md["plan_obj"], qd[l],
                                       k_new=knd[l], v_new=vnd[l], softmax_scale=scale,
                                       out=p2p.local_out(l).permute(1, 0, 2), peer_outs=p2p.peer_outs(l),
                                       ws=wsb, pdl=True, kv_early=True,
                                       multicast=getattr(p2p, "multicast", False), **gm)
                else:
                    bkv.decode_planned(pools[l], md["bt"], md["dirs"], md["lens"], md["plan_obj"], qd[l],
                                       k_new=knd[l], v_new=vnd[l], softmax_scale=scale,
                                       out=ol[l].permute(1, 0, 2), ws=wsb, pdl=True, kv_early=True, **gm)
                launches += 2                                  # decode kernel + cross-CTA merge kernel
                if tp > 1 and not attn_only and p2p is None and args.gather == "layer":
                    gather_heads(ol[l], og[l])
        if tp > 1 and not attn_only:
            if p2p is not None:
                p2p.barrier()
                launches += 1
            elif args.gather == "step":
                # a6: head-sharded TP needs no per-layer reassembly (each rank's o_proj shard
                # consumes its own heads); the step's outputs of every layer are reassembled
                # by ONE all-gather
                gather_heads(ol.view(n_layers * Hq, B, d), og.view(tp * n_layers * Hq, B, d))
            elif gather_only:
                for l in range(n_layers):
                    gather_heads(ol[l], og[l])
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

    p2p0 = p2ps[0] if p2ps else None
    full = lambda: step(meta_d, q_d, kn_d, vn_d, out_loc, out_glob, p2p0)
    attn = lambda: step(meta_d, q_d, kn_d, vn_d, out_loc, out_glob, p2p0, attn_only=True)
    gath = lambda: step(meta_d, q_d, kn_d, vn_d, out_loc, out_glob, p2p0, gather_only=True)

    # ---- eager warm-up, then capture the step (and attention-only / gather-only parts) in graphs
    for _ in range(args.warmup):
        launches_per_step = full()
    barrier()
    g_step, g_attn, g_gath = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    if args.graphs:
        try:
            with torch.cuda.graph(g_step):
                full()
            with torch.cuda.graph(g_attn):
                attn()
            if tp > 1 and p2p0 is None:
                with torch.cuda.graph(g_gath):
                    gath()
        except Exception as e:   # e.g. a collective that cannot be captured: time the eager launches
            print(f"bench: CUDA graph capture failed ({type(e).__name__}: {e}); running eagerly",
                  file=sys.stderr, flush=True)
            torch.cuda.synchronize(dev)
            args.graphs = False
    run_step = g_step.replay if args.graphs else full
    run_attn = g_attn.replay if args.graphs else attn
    run_gath = g_gath.replay if args.graphs else gath
    for _ in range(args.warmup):
        run_step()
    barrier()

    def timed(fn, n):
        """n back-to-back calls bracketed by barrier + sync; per-call events for percentiles.
        Returns (total ms max over ranks, per-call ms list of this rank)."""
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        barrier()
        evs[0].record(stream)
        for i in range(n):
            fn()
            evs[i + 1].record(stream)
        barrier()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
        return max_over_ranks(evs[0].elapsed_time(evs[n])), per

    # ---- device-resident timed region (W warm-up steps done above)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)                          # let nvidia-smi attach before the timed region
    ms_total, per_step = timed(run_step, args.steps)
    ms_step = ms_total / args.steps
    launches = launches_per_step * args.steps
    # ---- the hot path alone (decode + merge kernels of every layer, no reassembly), same stream
    for _ in range(2):
        run_attn()
    att_total, att_per = timed(run_attn, args.steps)
    att_avg_us = att_total * 1e3 / (args.steps * n_layers)
    gath_ms = None
    if tp > 1 and p2p0 is None:
        for _ in range(2):
            run_gath()
        gath_ms = timed(run_gath, args.steps)[0] / args.steps

    # ---- end to end through the public API: every step the host rebuilds the step's plan
    # (bkv_decode_plan), pinned host inputs go to the device, the step runs, outputs come back
    sets = []
    for si in range(n_sets):
        if si == 0:
            md, qd, knd, vnd, ol, og = meta_d, q_d, kn_d, vn_d, out_loc, out_glob
        else:
            md = dev_meta()
            qd, knd, vnd = torch.empty_like(q_d), torch.empty_like(kn_d), torch.empty_like(vn_d)
            qd.copy_(q_d), knd.copy_(kn_d), vnd.copy_(vn_d)
            ol = torch.empty_like(out_loc)
            og = p2ps[si].glob if p2ps else (torch.empty_like(out_glob) if out_glob is not None else None)
        p2p = p2ps[si] if p2ps else None
        fn = (lambda md=md, qd=qd, knd=knd, vnd=vnd, ol=ol, og=og, p2p=p2p: step(md, qd, knd, vnd, ol, og, p2p))
        g = torch.cuda.CUDAGraph() if args.graphs else None
        if si > 0:
            fn()                                          # eager warm-up of this set
            torch.cuda.synchronize(dev)
            if g is not None:
                with torch.cuda.graph(g):
                    fn()
        src = og if tp > 1 else ol
        sets.append({"md": md, "q": qd, "kn": knd, "vn": vnd, "run": (g_step.replay if si == 0 else g.replay)
                     if args.graphs else fn, "src": src,
                     "plan_h": torch.empty_like(meta_h["plan"]).pin_memory()})
    up = torch.cuda.Stream(dev)     # host -> device (one copy engine) ...
    down = torch.cuda.Stream(dev)   # ... and device -> host (the other), concurrently
    ev_h2d = [torch.cuda.Event() for _ in range(n_sets)]
    ev_comp = [torch.cuda.Event() for _ in range(n_sets)]
    ev_d2h = [torch.cuda.Event() for _ in range(n_sets)]
    h2d_bytes = [0]

    def h2d(si):
        s = sets[si]
        ev_h2d[si].synchronize()                          # this set's pinned plan buffer is free again
        hp = host_plan()                                  # the host scheduler's plan of this step
        used = bkv.plan_used_bytes(hp)
        s["plan_h"][:used].copy_(torch.from_numpy(hp.view(np.uint8)[:used]))
        with torch.cuda.stream(up):
            n = 0
            for k, v in meta_h.items():
                if k == "plan":                           # the plan's used bytes (fixed layout, entries last)
                    s["md"][k][:used].copy_(s["plan_h"][:used], non_blocking=True)
                    n += used
                    continue
                s["md"][k].copy_(v, non_blocking=True)
                n += v.numel() * v.element_size()
            for dst, srcv in ((s["q"], q_h), (s["kn"], kn_h), (s["vn"], vn_h)):
                dst.copy_(srcv, non_blocking=True)
                n += srcv.numel() * srcv.element_size()
            ev_h2d[si].record(up)
        h2d_bytes[0] = n

    def run_pipeline(n):
        up.wait_stream(stream)
        down.wait_stream(stream)
        h2d(0)
        for i in range(n):
            si = i % n_sets
            stream.wait_event(ev_h2d[si])
            # set si is rewritten by step i: step i - n_sets's outputs must be on the host.  p2p:
            # the PEERS write it as soon as they pass our barrier of step i-1, so that D2H must
            # be done before our step i-1 (i.e. wait for step i+1-n_sets's D2H here)
            j = i + 1 - n_sets if p2ps else i - n_sets
            if j >= 0:
                stream.wait_event(ev_d2h[j % n_sets])
            sets[si]["run"]()
            ev_comp[si].record(stream)
            if i + 1 < n:                                  # inputs of step i+1 overlap step i
                sj = (i + 1) % n_sets
                if i + 1 >= n_sets:
                    up.wait_event(ev_comp[sj])
                h2d(sj)
            with torch.cuda.stream(down):                  # outputs of step i overlap step i+1
                down.wait_event(ev_comp[si])
                out_h.copy_(sets[si]["src"], non_blocking=True)
                ev_d2h[si].record(down)
        stream.wait_stream(up)
        stream.wait_stream(down)

    run_pipeline(2)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run_pipeline(args.steps)
    e1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    for p in (p2ps or []):
        p.check()
    clk = clocks.stop()                      # clocks sampled over every timed region
    d2h = out_h.numel() * 2

    peak, peak_src = load_peaks()
    shards = None
    if ws == 1 and not args.no_shards:
        shards = measure_shards(dev, peak, args.seed)
    if rank != 0:
        dist.destroy_process_group()
        return
    alg_bytes, kv_bytes = algorithmic_bytes(lay, H, Hq, d, bs)
    alg_bytes += append_bytes(B, H, d)   # the fused step also reads the new rows and writes them into the pool
    achieved = alg_bytes / (att_avg_us * 1e-6) / 1e9
    static = meta_d["plan_obj"].header["P"] < PLANNED_DYNAMIC_P
    tok_s = B / (ms_step * 1e-3)
    cpu = cpu_baseline(args, lay, sh, n_layers) if (ws == 1 and not args.no_cpu) else None
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
        "config": workload_config(args, ws, sh, lay),
        "step_ms": {"mean": ms_step, "median": statistics.median(per_step), "p10": pct(per_step, 10),
                    "p90": pct(per_step, 90), "n": len(per_step)},
        "detail": {
            "kv_heads_per_gpu": H, "q_heads_per_gpu": Hq,
            "mean_ctx": float(lay.lens.mean()), "max_ctx": int(lay.lens.max()),
            "shared_blocks": int(lay.n_shared),
            "kv_mb_per_layer_per_gpu": kv_bytes / 1e6,
            "per_layer_us": ms_step * 1e3 / n_layers,
            "attn_us_per_layer": att_avg_us,
            "attn_us_per_layer_pct": {"median": statistics.median(att_per) * 1e3 / n_layers,
                                      "p10": pct(att_per, 10) * 1e3 / n_layers,
                                      "p90": pct(att_per, 90) * 1e3 / n_layers},
            "attn_share_of_step": att_avg_us * n_layers / (ms_step * 1e3),
            "reassembly_ms_per_step": gath_ms,
            "cuda_graphs": bool(args.graphs),
            "path": "bkv_decode_plan once per step (host) + bkv_decode_planned per layer (fused append, "
                    "PDL, early KV tiles)",
            "plan_blocks_per_warp": meta_d["plan_obj"].header["P"],
            "reassembly": ("nvls multicast stores + peer barrier (bkv_decode_planned, BKV_FLAG_PEER_MULTICAST)"
                           if p2ps and args.reassembly == "nvls"
                           else "p2p stores + peer barrier (bkv_decode_planned peer_outs)" if p2ps
                           else f"nccl all_gather_into_tensor, one per {args.gather}" if tp > 1
                           else "none (1 GPU)"),
            "attn_layer_tokens_per_s": B / (att_avg_us * 1e-6),
        },
        "roofline": {
            "bound": "hbm",
            "kernel": ("bkv::planned_kernel + planned_xmerge_kernel (static plan)" if static else
                       "bkv::decode_kernel + merge_kernel (dynamic schedule: plan ranges >= "
                       f"{PLANNED_DYNAMIC_P} blocks per warp)") + ", one layer, fused append",
            "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak, "algorithmic_bytes_per_launch": alg_bytes,
            "traffic": ncu_traffic(f"{args.config}_tp{tp}"),
            "traffic_source": "profiles/r02/ncu_traffic.json (ncu --set full of these kernels on this shard; "
                              "not measured in this run)",
        },
        "shards": shards,
        "cpu_baseline": cpu,
        "e2e": {"value": B / (ms_e2e * 1e-3), "unit": "tokens/s", "ms_per_step": ms_e2e,
                "pipeline": f"host rebuilds the step's plan; {n_sets} buffer sets; one copy stream uploads "
                            f"step i+1 while step i computes, another downloads step i's outputs",
                "h2d_bytes_per_step": int(h2d_bytes[0]), "d2h_bytes_per_step": int(d2h)},
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
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline (oracle) leg")
    ap.add_argument("--no-shards", action="store_true", help="skip the per-shard table (N = 1)")
    ap.add_argument("--general-map", action="store_true",
                    help="FindBlock-style general block map (partly filled entries, SURVEY §8(f) f3)")
    ap.add_argument("--gather", default="step", choices=["step", "layer"],
                    help="N>1, nccl reassembly: one all-gather per step of every layer's outputs (default) "
                         "or one per layer")
    ap.add_argument("--reassembly", default="nccl", choices=["nccl", "p2p", "nvls"],
                    help="N>1: NCCL all-gather (default), fused NVLink stores (CUDA IPC peer memory) or "
                         "fused NVLS multicast stores (torch symmetric memory's multicast mapping)")
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

"""Summarise round r02's ncu captures (scripts/profile_r02.sh) into profiles/r02/.

Writes profiles/r02/launches_<cfg>.csv (per-kernel shares of the bench step),
profiles/r02/ncu_summary.md and profiles/r02/ncu_traffic.json (DRAM bytes of one
layer's kernels per shard, read by bench.py as roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof_r02")
DST = os.environ.get("BKV_SUMMARY_DST", os.path.join(ROOT, "profiles", "r02"))
os.makedirs(DST, exist_ok=True)
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from synth import CONFIGS, make_case  # noqa: E402
from synth.workload import shard_heads  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
KERNELS = ("planned_xmerge_kernel", "planned_kernel", "decode_kernel", "merge_kernel", "kv_append_kernel",
           "prefill_tc_kernel", "prefill_kernel", "peer_barrier_kernel")


def short(name):
    for k in KERNELS:
        if k in name:
            return "bkv::" + k + name[name.index(k) + len(k):].split("(")[0]
    return name.split("(")[0][:60]


def launch_list(fname):
    path = os.path.join(SRC, fname)
    if not os.path.exists(path):
        return None
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    fam = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        f = short(r[iN])
        fam[f][0] += 1
        fam[f][1] += float(r[iV]) / 1e3
    return fam


def alg_bytes(cfg, tp):
    """bench.py's algorithmic bytes of one layer (KV, q/out, map, lengths) + the fused append."""
    sh = CONFIGS[cfg]
    lay = make_case(cfg, 0).layout
    kv, q = shard_heads(sh, tp, 0)
    L = lay.lens.astype(np.int64)
    nb = (L + sh.block_size - 1) // sh.block_size
    H, Hq, d, B = len(kv), len(q), sh.head_dim, lay.batch
    return float(L.sum()) * 4 * H * d + 4.0 * B * Hq * d + nb.sum() * 5 + 4 * B + 8.0 * B * H * d


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "Kernel Name"]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}


def read_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hh, uu = r[0], r[1]
    rows = []
    for vv in r[2:]:
        m = {n: vv[i] for i, n in enumerate(hh) if n in WANT}
        u = {n: uu[i] for i, n in enumerate(hh) if n in WANT}
        val = lambda k: float(m.get(k, 0) or 0) * SCALE.get(u.get(k, ""), 1.0)
        rows.append({"kernel": short(m.get("Kernel Name", "?")), "dur_us": val("gpu__time_duration.sum"),
                     "dram_mb": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                     "dram_pct": m.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ""),
                     "sm_pct": m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", ""),
                     "issue_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", ""),
                     "regs": m.get("launch__registers_per_thread", ""),
                     "tensor_pct": m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "")})
    return rows


md = ["# ncu summary, round r02", "",
      "`scripts/profile_r02.sh`: ncu --set full --clock-control none, cold L2 (ncu's default cache",
      "control), each kernel serialised and timed ALONE.  One layer of the planned decode = the",
      "decode kernel (append fused in) + the cross-CTA merge kernel.  `alg MB` = bench.py's",
      "algorithmic bytes of the layer incl. the fused append; `frac` = alg bytes / the layer's ncu",
      f"time (decode + merge) / the measured {PEAK:.0f} GB/s copy peak (MEASURED_PEAKS.json).", "",
      "| shard | kernel | dur us | dram MB | dram % peak | SM % | issue % | regs |",
      "|---|---|---|---|---|---|---|---|"]
layer = []
traffic = {}
prefill = []
for fn in sorted(os.listdir(SRC)) if os.path.isdir(SRC) else []:
    if not fn.endswith(".ncu-rep"):
        continue
    name = fn[:-8]
    rows = read_rep(os.path.join(SRC, fn))
    for r in rows:
        md.append(f"| {name} | {r['kernel']} | {r['dur_us']:.1f} | {r['dram_mb']:.1f} | {r['dram_pct']} | "
                  f"{r['sm_pct']} | {r['issue_pct']} | {r['regs']} |")
    if name.startswith(("planned_", "dynamic_")) and rows:
        cfg, tp = name.split("_", 1)[1].rsplit("_tp", 1)
        tp = int(tp)
        alg = alg_bytes(cfg, tp) / 1e6
        # one layer = one launch of each kernel; captures hold several layers: mean per kernel
        per = defaultdict(list)
        for r in rows:
            per[r["kernel"]].append(r)
        mean = lambda k, f: sum(x[f] for x in per[k]) / len(per[k])
        dur = sum(mean(k, "dur_us") for k in per)
        dram = sum(mean(k, "dram_mb") for k in per)
        main_k = rows[0]["kernel"]
        layer.append((f"{cfg} tp{tp}", name.split("_")[0], mean(main_k, "dur_us"), dur, dram, alg,
                      alg / dur * 1e3 / PEAK, len(per[main_k])))
        traffic[f"{cfg}_tp{tp}"] = dram * 1e6   # per layer (mean over the captured layers)
    if name.startswith("prefill_") and rows:
        cfg = name[len("prefill_"):].rsplit("_tp", 1)[0]
        sh = CONFIGS[cfg]
        lay = make_case(cfg, 0).layout
        rng = np.random.default_rng(1)
        be = np.flatnonzero(lay.is_be)
        pre = rng.choice(be, size=min(16, be.size), replace=False)
        Lp = lay.lens[pre].astype(np.int64)
        flops = 4.0 * sh.head_dim * sh.num_q_heads * float((Lp * (Lp + 1) // 2).sum())
        r = rows[0]
        prefill.append(f"| {name} | {r['dur_us']:.1f} | {flops / 1e9:.1f} | "
                       f"{flops / (r['dur_us'] * 1e-6) / 1e12:.1f} | {r['tensor_pct']} |")
md += ["", "## Per-layer roofline from ncu (kernels timed alone)", "",
       "| shard | path | layers | decode kernel us | layer us (decode + merge) | dram MB | alg MB | dram/alg | frac of measured peak |",
       "|---|---|---|---|---|---|---|---|---|"]
for s, path, dk, dur, dram, alg, frac, nl in layer:
    md.append(f"| {s} | {path} | {nl} | {dk:.1f} | {dur:.1f} | {dram:.1f} | {alg:.1f} | {dram / alg:.3f} | {frac:.3f} |")
if prefill:
    md += ["", "## Prefill kernel (tensor-bound; causal flops of the 16 whole-prompt prefills)", "",
           "| capture | dur us | GFLOP | TFLOP/s | tensor pipe % |", "|---|---|---|---|---|"] + prefill
for cfg, cmd in (("opt13b", "python bench.py --steps 2 --warmup 3 --no-cpu --no-shards"),
                 ("llama70b", "python bench.py --config llama70b --layers 8 --steps 2 --warmup 3 --no-cpu --no-shards")):
    fam = launch_list(f"launches_{cfg}.csv")
    if fam is None:
        continue
    ours = {k: v for k, v in fam.items() if k.startswith("bkv::")}
    tot = sum(v[1] for v in ours.values())
    with open(os.path.join(DST, f"launches_{cfg}.csv"), "w") as f:
        f.write("kernel,launches,total_us,mean_us,share_of_bkv_time\n")
        for k, (n, t) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k},{n},{t:.1f},{t / n:.2f},{(t / tot if k in ours else 0):.4f}\n")
    md += ["", f"## Launch list of `{cmd}` ({cfg}, 1 GPU)", "",
           "ncu --metrics gpu__time_duration.sum --clock-control none; serialised, cold-ish: compare SHARES.", "",
           "| kernel | launches | total us | mean us | share of bkv time |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        if k in ours:
            md.append(f"| {k} | {n} | {t:.0f} | {t / n:.1f} | {t / tot:.3f} |")
    others = {k: v for k, v in fam.items() if k not in ours}
    if others:
        md.append(f"| (not ours: {', '.join(sorted(others))}) | {sum(v[0] for v in others.values())} | "
                  f"{sum(v[1] for v in others.values()):.0f} | | |")
open(os.path.join(DST, "ncu_summary.md"), "w").write("\n".join(md) + "\n")
json.dump(traffic, open(os.path.join(DST, "ncu_traffic.json"), "w"), indent=1)
print("\n".join(md))

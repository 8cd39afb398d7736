"""Summarise a round's ncu captures into profiles/ (committed evidence).

usage: python scripts/summarize_profiles.py r01
Reads gpurun_out/prof_<r>/ ; writes profiles/<r>_launches.csv (per-kernel
shares of the bench step), profiles/<r>_ncu_summary.md and profiles/ncu_traffic.json.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

R = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", f"prof_{R}")
DST = os.path.join(ROOT, "profiles")
os.makedirs(DST, exist_ok=True)


def short(name):
    for k in ("decode_kernel", "merge_kernel", "kv_append_kernel", "kv_append_general_kernel", "slot_copy_kernel",
              "prefill_tc_kernel", "prefill_kernel", "peer_barrier_kernel"):
        if k in name:
            return "bkv::" + k + name[name.index(k) + len(k):].split("(")[0]
    return name.split("(")[0][:60]


# ---- 1. launch lists of the bench commands: time per kernel family and share
def launch_list(fname):
    path = os.path.join(SRC, fname)
    if not os.path.exists(path):
        return None, None, 0.0
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    fam = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        f = short(r[iN])
        fam[f][0] += 1
        fam[f][1] += float(r[iV]) / 1e3
    ours = {k: v for k, v in fam.items() if k.startswith("bkv::")}
    return fam, ours, sum(v[1] for v in ours.values())


lists = {}
for cfg in ("opt13b", "llama70b"):
    fam, ours, tot = launch_list(f"launches_{cfg}.csv")
    if fam is None:
        continue
    lists[cfg] = (fam, ours, tot)
    with open(os.path.join(DST, f"{R}_launches{'' if cfg == 'opt13b' else '_' + cfg}.csv"), "w") as f:
        f.write("kernel,launches,total_us,mean_us,share_of_bkv_time\n")
        for k, (n, t) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k},{n},{t:.1f},{t / n:.2f},{(t / tot if k in ours else 0):.4f}\n")

# ---- 2. full captures
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
traffic = {}
md = [f"# ncu summary, round {R}", "",
      "Captured with `scripts/profile_round.sh` (ncu --set full --clock-control none, one decode",
      "launch after warm-up, cold L2 per ncu's default cache control).  `alg MB` = algorithmic",
      "bytes of the launch (bench.py definition); `dram MB` = dram__bytes_read + write.", ""]
md.append("| capture | dur us | dram MB | alg MB | dram/alg | dram TB/s | dram % peak | SM % | issue % | regs | tensor % |")
md.append("|---|---|---|---|---|---|---|---|---|---|---|")
sys.path.insert(0, ROOT)
import numpy as np
from synth import CONFIGS, make_case
from synth.workload import shard_heads


def alg_bytes(cfg, tp):
    sh = CONFIGS[cfg]
    lay = make_case(cfg, 0).layout
    kv, q = shard_heads(sh, tp, 0)
    L = lay.lens.astype(np.int64)
    nb = (L + sh.block_size - 1) // sh.block_size
    return float(L.sum()) * 4 * len(kv) * sh.head_dim + 4.0 * lay.batch * len(q) * sh.head_dim + nb.sum() * 5 + 4 * lay.batch


prefill_lines = []
for fn in sorted(os.listdir(SRC)):
    if not fn.endswith(".ncu-rep"):
        continue
    out = subprocess.run(["ncu", "-i", os.path.join(SRC, fn), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        continue
    hh, uu, vv = r[0], r[1], r[2]
    m = {n: vv[i] for i, n in enumerate(hh) if n in WANT}
    units = {n: uu[i] for i, n in enumerate(hh) if n in WANT}
    SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
             "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    def val(k, dflt=0.0):
        return float(m.get(k, dflt)) * SCALE.get(units.get(k, ""), 1.0)
    dur_us = val("gpu__time_duration.sum")
    dram_mb = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    name = fn[:-8]
    alg = None
    if name.startswith("decode_"):
        cfg, tp = name[len("decode_"):].rsplit("_tp", 1)
        alg = alg_bytes(cfg, int(tp)) / 1e6
        traffic[f"{cfg}_tp{tp}"] = dram_mb * 1e6
    md.append(f"| {name} | {dur_us:.1f} | {dram_mb:.1f} | {alg if alg is None else round(alg, 1)} | "
              f"{'' if alg is None else round(dram_mb / alg, 3)} | {dram_mb / dur_us:.2f} | "
              f"{m.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', m.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', ''))} | "
              f"{m.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', '')} | "
              f"{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', '')} | "
              f"{m.get('launch__registers_per_thread', '')} | "
              f"{m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', '')} |")
    if name.startswith("prefill_"):
        # the bench_prefill --no-decodes workload: 16 BE requests prefilling their whole prompt
        cfg = name[len("prefill_"):].rsplit("_tp", 1)[0]
        sh = CONFIGS[cfg]
        lay = make_case(cfg, 0).layout
        rng = np.random.default_rng(1)
        be = np.flatnonzero(lay.is_be)
        pre = rng.choice(be, size=min(16, be.size), replace=False)
        Lp = lay.lens[pre].astype(np.int64)
        flops = 4.0 * sh.head_dim * sh.num_q_heads * float((Lp * (Lp + 1) // 2).sum())
        prefill_lines.append(f"| {name} | {dur_us:.1f} | {flops / 1e9:.1f} | {flops / (dur_us * 1e-6) / 1e12:.1f} | "
                             f"{m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', '')} |")
if prefill_lines:
    md += ["", "## Prefill kernel (tensor-bound; causal flops of the 16 whole-prompt prefills)", "",
           "| capture | dur us | GFLOP | TFLOP/s | tensor pipe % |", "|---|---|---|---|---|"] + prefill_lines
for cfg, (fam, ours, tot) in lists.items():
    cmd = "python bench.py --steps 2 --warmup 3 --no-cpu" if cfg == "opt13b" else \
        "python bench.py --config llama70b --layers 8 --steps 2 --warmup 3 --no-cpu"
    md += ["", f"## Launch list of `{cmd}` ({cfg}, 1 GPU)", "",
           "ncu --metrics gpu__time_duration.sum --clock-control none; serialised, cold-ish: compare SHARES.", "",
           "| kernel | launches | total us | mean us | share of bkv time |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        if k in ours:
            md.append(f"| {k} | {n} | {t:.0f} | {t / n:.1f} | {t / tot:.3f} |")
open(os.path.join(DST, f"{R}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
json.dump(traffic, open(os.path.join(DST, "ncu_traffic.json"), "w"), indent=1)
print("\n".join(md))

"""Dev: aggregate ncu SASS-level warp-stall samples by CUDA source line.

usage: python scripts/ncu_lines.py <report.ncu-rep> <kernel-mangled-name> [top]
Needs libbkv.so built with -lineinfo (nvdisasm --print-line-info).
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2504_09590_b200", "libbkv.so")],
               cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("decode_attention")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith(f".text.{kname}:")][0]
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        break
    m = re.search(r'//## File ".*?([^/]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        off2line[int(m.group(1), 16)] = (cur, m.group(2).split(";")[0].strip())
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
addrs = [int(r[0], 16) for r in data]
base = min(addrs)
agg = defaultdict(lambda: [0, 0, ""])
tot = 0
for r in data:
    off = int(r[0], 16) - base
    ln, ins = off2line.get(off, ("?", ""))
    sm = int(r[iS]) if r[iS].isdigit() else 0
    ex = int(r[iE]) if r[iE].isdigit() else 0
    a = agg[ln]
    a[0] += sm
    a[1] = max(a[1], ex)
    if not a[2]:
        a[2] = ins
    tot += sm
src = open(os.path.join(ROOT, "paper_2504_09590_b200", "csrc", "decode_attention.cu")).read().splitlines()
print(f"total samples {tot}")
for ln, (sm, ex, ins) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    text = ""
    if ln and ln.startswith("decode_attention.cu:"):
        n = int(ln.split(":")[1])
        text = src[n - 1].strip()[:70] if n - 1 < len(src) else ""
    print(f"{sm:6d} {100.0 * sm / max(tot, 1):5.1f}%  exec {ex:8d}  {ln:26s} {text}")

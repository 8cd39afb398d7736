"""Summarise an ncu report: key raw metrics + top SASS stall sites."""
import csv, subprocess, sys, io
def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
            'sm__cycles_elapsed.avg.per_second']
    d = {}
    for i, n in enumerate(h):
        if n in want: d[n] = (v[i], u[i])
    return d
def sass(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]; data = rows[2:]
    iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
    tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
    res = [f"total stall samples {tot}"]
    for r in sorted(data, key=lambda r: -int(r[iS]) if r[iS].isdigit() else 0)[:top]:
        res.append(f"{r[iS]:>6} {r[iE]:>9}  {r[0][-5:]}  {r[1][:80]}")
    return res
if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        for k, (v, u) in raw(rep).items(): print(f"  {k} = {v} {u}")
        for l in sass(rep, 25): print("  " + l)

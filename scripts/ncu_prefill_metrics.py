"""Key metrics of one `ncu --set full` capture of the tcgen05 prefill kernel, from its
`ncu -i ... --page raw --csv` export (scripts/round_evidence.sh, prefill step).

    python scripts/ncu_prefill_metrics.py raw.csv > profiles/r02/prefill_ncu.txt
"""
import csv
import sys

KEYS = ("Kernel Name", "gpu__time_duration.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_writes_op_stt.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size")

rows = list(csv.reader(open(sys.argv[1])))
head, units, vals = rows[0], rows[1], rows[2]
print("ncu --set full --clock-control none of bkv::prefill_tc_kernel<2>: Llama-70B TP1, 16 whole-prompt "
      "prefills (174.9 GFLOP causal), one launch timed alone")
for k in KEYS:
    if k in head:
        i = head.index(k)
        print(f"{k} = {vals[i]} {units[i]}".rstrip())

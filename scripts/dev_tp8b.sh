#!/bin/bash
# Dev: ncu source-level capture of the Llama-70B TP8 planned kernel + a finer prefetch sweep.
set -x
cd ${GRAFT_REPO_ROOT:-.}; O=gpurun_out/dev; mkdir -p $O
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
SH="llama70b:8:planned_early opt13b:8:planned_early llama70b:4:planned_early"
for PF in 2 3 4 5 6; do
  BKV_PLANNED_XMW=0 BKV_PLANNED_PF=$PF timeout 300 python scripts/quick_perf.py $SH 2>&1 | sed "s/^/pf$PF /"
done | tee $O/tp8_pf.txt
BKV_PLANNED_XMW=0 BKV_PLANNED_PF=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:planned_kernel -s 12 -c 1 \
   -o $O/planned_llama70b_tp8 python scripts/ncu_target_planned.py llama70b 8 16 > $O/ncu_log.txt 2>&1
ncu -i $O/planned_llama70b_tp8.ncu-rep --page source --csv --print-source sass > $O/planned_tp8_source.csv 2>&1
ncu -i $O/planned_llama70b_tp8.ncu-rep --page raw --csv > $O/planned_tp8_raw.csv 2>&1
ls -la $O

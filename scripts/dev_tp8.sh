#!/bin/bash
# Dev (not evidence): small-shard decode experiments on one GPU.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out/dev
O=gpurun_out/dev
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
SH="llama70b:8:planned_early opt13b:8:planned_early llama70b:4:planned_early opt13b:2:planned_early llama70b:1:planned_early"
for cfg in "4 0" "4 2" "4 3" "4 4" "2 2" "2 3" "0 3" "3 3"; do set -- $cfg
  BKV_PLANNED_XMW=0 BKV_PLANNED_PF=$1 BKV_PLANNED_PFD=$2 timeout 300 python scripts/quick_perf.py $SH 2>&1 | sed "s/^/pf$1 pfd$2 /"
done | tee $O/tp8_pfd.txt

#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out/dev
python paper_2504_09590_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_planned_gpu.py -x -q 2>&1 | tail -3 | tee gpurun_out/dev/planned_tests.txt
SH="llama70b:8:planned_early opt13b:8:planned_early llama70b:4:planned_early opt13b:4:planned_early llama70b:2:planned_early opt13b:2:planned_early llama70b:1:planned_early opt13b:1:planned_early opt30b:4:planned_early"
for PF in 4 3; do BKV_PLANNED_PF=$PF timeout 600 python scripts/quick_perf.py $SH 2>&1 | sed "s/^/pf$PF /"; done | tee gpurun_out/dev/perf.txt

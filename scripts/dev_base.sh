set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
python scripts/quick_perf.py llama70b:1:fused llama70b:2:fused llama70b:4:fused llama70b:8:fused opt13b:1:fused opt13b:2:fused opt13b:4:fused opt13b:8:fused opt30b:4:fused 2>&1 | tee gpurun_out/base_perf.txt
BKV_BUILD_TRACE=1 python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
for s in "llama70b 8" "llama70b 4" "opt13b 8"; do python scripts/trace_run.py $s; done 2>&1 | tee gpurun_out/base_trace.txt
python paper_2504_09590_b200/build.py --force > /dev/null 2>&1

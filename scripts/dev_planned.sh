set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
BKV_PLANNED_WARPS=12 timeout 900 python -m pytest tests/test_planned_gpu.py -x -q -k "small or geometries or edge or general_map or fused_step or llama70b-8-0 or opt13b-1-0 or graph" 2>&1 | tail -3 | tee gpurun_out/planned_tests.txt
for W in 8 12 10; do BKV_PLANNED_WARPS=$W timeout 600 python scripts/quick_perf.py llama70b:8:planned_early llama70b:4:planned_early llama70b:2:planned_early llama70b:1:planned_early opt13b:8:planned_early opt13b:4:planned_early opt13b:1:planned_early opt30b:4:planned_early 2>&1; done | tee gpurun_out/planned_perf.txt

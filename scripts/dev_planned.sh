set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
timeout 900 python -m pytest tests/test_planned_gpu.py -x -q -k "not sweep and not full_size" 2>&1 | tail -3 | tee gpurun_out/planned_tests.txt
BKV_PLANNED_SLOTS=3 timeout 900 python -m pytest tests/test_planned_gpu.py -x -q -k "small or llama70b-8-0 or geometries" 2>&1 | tail -3 | tee -a gpurun_out/planned_tests.txt
for S in 2 3; do BKV_PLANNED_SLOTS=$S timeout 600 python scripts/quick_perf.py llama70b:8:planned_early llama70b:4:planned_early llama70b:1:planned_early opt13b:8:planned_early opt13b:1:planned_early 2>&1; done | tee gpurun_out/planned_perf.txt

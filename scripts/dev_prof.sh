set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
timeout 1500 python -m pytest tests/test_planned_gpu.py -x -q 2>&1 | tail -3 | tee gpurun_out/prof_tests.txt
timeout 1500 bash scripts/profile_r02.sh > gpurun_out/prof_r02.log 2>&1
timeout 600 python bench.py --config opt30b --no-shards --no-cpu > gpurun_out/bench_opt30b.json 2>> gpurun_out/bench_err.txt

set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
timeout 900 python -m pytest tests/test_planned_gpu.py -x -q -k "graph or small" 2>&1 | tail -3 | tee gpurun_out/bench_tests.txt
timeout 900 python bench.py > gpurun_out/bench_opt13b.json 2> gpurun_out/bench_err.txt; tail -3 gpurun_out/bench_err.txt
timeout 900 python bench.py --config llama70b --no-shards --no-cpu > gpurun_out/bench_llama70b.json 2>> gpurun_out/bench_err.txt
timeout 900 python bench.py --config opt30b --no-shards --no-cpu > gpurun_out/bench_opt30b.json 2>> gpurun_out/bench_err.txt
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench_err.txt
bash scripts/n2_smoke.sh 2>&1 | tee gpurun_out/n2_smoke.txt
timeout 900 python -m pytest tests/test_bench_contract.py -x -q 2>&1 | tail -3 | tee -a gpurun_out/bench_tests.txt

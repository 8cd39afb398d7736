python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r20
timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q > gpurun_out/r20/pytest_prefill.log 2>&1; echo "exit $?" >> gpurun_out/r20/pytest_prefill.log
for a in "--config llama70b --tp 1" "--config llama70b --tp 1 --no-decodes" "--config llama70b --tp 8" "--config opt13b --tp 2"; do
  timeout 300 python scripts/bench_prefill.py $a 2>&1 | tail -n1 >> gpurun_out/r20/tc.jsonl
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r20/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r20/pytest.log
bash scripts/sanitize.sh r20

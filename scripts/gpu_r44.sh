python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r44
timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q > gpurun_out/r44/pytest_qt1.log 2>&1; echo "exit $?" >> gpurun_out/r44/pytest_qt1.log
BKV_PREFILL_QT=2 timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q > gpurun_out/r44/pytest_qt2.log 2>&1; echo "exit $?" >> gpurun_out/r44/pytest_qt2.log
for qt in 1 2; do
for a in "--config llama70b --tp 1" "--config llama70b --tp 1 --no-decodes" "--config llama70b --tp 8" "--config opt13b --tp 2"; do BKV_PREFILL_QT=$qt timeout 300 python scripts/bench_prefill.py $a 2>&1 | tail -n1 | sed "s/^/$qt /" >> gpurun_out/r44/tc.txt; done
done

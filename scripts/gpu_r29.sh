python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r29
BKV_FUSED_MERGE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fused_step.py tests/test_general_map_gpu.py -x -q > gpurun_out/r29/pytest_fused.log 2>&1; echo "exit $?" >> gpurun_out/r29/pytest_fused.log
for c in llama70b:1:fused llama70b:8:fused llama70b:4:fused llama70b:2:fused opt13b:1:fused opt13b:8:fused opt30b:1:fused; do
  for fm in 0 1; do BKV_FUSED_MERGE=$fm timeout 120 python scripts/quick_perf.py $c 2>&1 | tail -n1 | sed "s/^/FM=$fm /" >> gpurun_out/r29/merge.txt; done
done

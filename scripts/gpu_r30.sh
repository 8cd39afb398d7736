python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r30
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r30/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r30/pytest.log
for c in llama70b:8:fused opt13b:8:fused llama70b:4:fused opt13b:2:fused opt13b:1:fused llama70b:1:fused opt30b:1:fused; do
  for kv in 0 1; do BKV_KV_COMBINED=$kv timeout 120 python scripts/quick_perf.py $c 2>&1 | tail -n1 | sed "s/^/KV=$kv /" >> gpurun_out/r30/kv.txt; done
done

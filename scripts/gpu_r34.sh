python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r34
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r34/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r34/pytest.log
for c in llama70b:1:fused llama70b:8:fused llama70b:4:fused opt13b:1:fused opt13b:8:fused opt30b:1:fused; do
  for pr in 1 0; do BKV_MERGE_PER_ROW=$pr timeout 120 python scripts/quick_perf.py $c 2>&1 | tail -n1 | sed "s/^/PERROW=$pr /" >> gpurun_out/r34/merge.txt; done
done

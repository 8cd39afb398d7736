python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r19
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r19/pytest.log 2>&1; echo "pytest $?" >> gpurun_out/r19/pytest.log
for c in llama70b:1:fused opt13b:1:fused opt30b:1:fused llama70b:8:fused opt13b:8:fused opt13b:2:fused llama70b:4:fused; do
  for sm in 0 1; do BKV_SEPARATE_MERGE=$sm timeout 120 python scripts/quick_perf.py $c 2>&1 | tail -n1 | sed "s/^/SEP=$sm /" >> gpurun_out/r19/merge.txt; done
done
bash scripts/sanitize.sh r19

python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r18
for a in "--config llama70b --tp 1" "--config llama70b --tp 1 --no-decodes" "--config llama70b --tp 8" "--config opt13b --tp 2"; do
  timeout 300 python scripts/bench_prefill.py $a 2>&1 | tail -n1 >> gpurun_out/r18/tc.jsonl
  BKV_PREFILL_MMA_SYNC=1 timeout 300 python scripts/bench_prefill.py $a 2>&1 | tail -n1 >> gpurun_out/r18/mmasync.jsonl
done
for c in llama70b:1:fused opt13b:1:fused llama70b:8:fused; do
  for dbg in 0 2; do BKV_DEBUG=$dbg timeout 120 python scripts/quick_perf.py $c 2>&1 | tail -n1 >> gpurun_out/r18/merge.txt; done
done
bash scripts/sanitize.sh r18

# dev: A/B of launch-level changes on the per-layer decode time (CUDA graph, PDL)
for dbg in 0 32 0 32; do
  BKV_DEBUG=$dbg python scripts/quick_perf.py llama70b:1:fused llama70b:8:fused opt13b:1:fused opt13b:4:fused 2>&1 | grep -v Warn
done

# dev: A/B of decode variants on the per-layer time (CUDA graph, PDL)
for env in "BKV_FUSED_MERGE=0" "BKV_FUSED_MERGE=1" "BKV_SMALL_PLAN=0" "BKV_UNITS_PER_WARP=2"; do
  echo "== $env"
  env $env python scripts/quick_perf.py llama70b:8:fused llama70b:4:fused opt13b:8:fused llama70b:1:fused 2>&1 | grep -v Warn
done

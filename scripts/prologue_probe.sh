for env in "BKV_FUSED_MERGE=0" "BKV_FUSED_MERGE=1"; do
  echo "== $env"
  env $env python scripts/quick_perf.py llama70b:8:fused llama70b:4:fused opt13b:8:fused llama70b:1:fused opt13b:1:fused 2>&1 | grep -v Warn
done

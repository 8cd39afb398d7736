set -x
python __graft_entry__.py >/dev/null 2>&1 || true
for env in "" "BKV_UNITS_PER_WARP=2" "BKV_UNITS_PER_WARP=4" "BKV_SLOTS=3" "BKV_MIN_SPLIT=24" "BKV_MIN_SPLIT=32" "BKV_SLOTS=3 BKV_UNITS_PER_WARP=2"; do
  echo "=== $env"
  env $env timeout 300 python scripts/quick_perf.py llama70b:1:fused llama70b:8:fused opt13b:1:fused opt13b:4:fused 2>&1 | grep -v Warn
done

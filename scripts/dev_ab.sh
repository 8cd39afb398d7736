cd ${GRAFT_REPO_ROOT:-.}
perf() { timeout 120 python scripts/bench_prefill.py --config llama70b --no-decodes 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'])"; }
echo "default: $(perf)"
echo "QT=1: $(BKV_PREFILL_QT=1 perf)"
for d in "-DBKV_POLY_PAIRS=0" "-DBKV_POLY_PAIRS=4" "-DBKV_POLY_PAIRS=1"; do
  BKV_BUILD_DEFINES="$d" python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
  echo "$d: $(perf)"
done

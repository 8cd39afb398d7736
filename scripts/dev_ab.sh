#!/bin/bash
# Dev (not evidence): A/B of compile-time prefill variants on one GPU.
#   bash scripts/dev_ab.sh "-DBKV_PINGPONG=1" ...   (each argument: one BKV_BUILD_DEFINES build)
cd ${GRAFT_REPO_ROOT:-.}
perf() {
  for a in "--no-decodes" "--tp 8"; do
    echo -n " $a: $(timeout 120 python scripts/bench_prefill.py --config llama70b $a 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'], 1))")"
  done
  echo
}
python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
echo "default:$(perf)"
for d in "$@"; do
  BKV_BUILD_DEFINES="$d" python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
  echo "$d:$(perf)"
  timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -1
done
python paper_2504_09590_b200/build.py --force > /dev/null 2>&1

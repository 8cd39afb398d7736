#!/bin/bash
# Dev (not evidence): prefill kernel parity + throughput on one GPU.
#   bash scripts/dev_prefill.sh [extra env assignments for an A/B run, e.g. BKV_PREFILL_Q_LDG=1]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out/dev; O=gpurun_out/dev
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
timeout 240 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -5 | tee $O/prefill_tests.txt
perf() {
  for a in "--no-decodes" "" "--tp 8"; do
    env "$@" timeout 120 python scripts/bench_prefill.py --config llama70b $a 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$* $a', {k: d[k] for k in ('value','unit')}, d.get('roofline',{}).get('frac'), d.get('detail',{}).get('prefill_tflops'))"
  done
}
perf X=1 | tee $O/prefill_perf.txt
for v in "$@"; do perf $v | tee -a $O/prefill_perf.txt; done

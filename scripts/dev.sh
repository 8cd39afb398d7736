#!/bin/bash
# Dev runs on ONE GPU under gpurun (not evidence; round evidence: scripts/round_evidence.sh).
#   bash scripts/dev.sh prefill [ENV=VAL ...]     prefill parity tests + throughput (plus one line per env A/B)
#   bash scripts/dev.sh ab "-DDEFINE=1" ...       compile-time A/B builds (BKV_BUILD_DEFINES) of the prefill kernel
#   bash scripts/dev.sh prefill-ncu               ncu --set full of the tcgen05 prefill kernel, exported on the box
#   bash scripts/dev.sh decode                    decode parity subset + quick per-shard timing
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out/dev; O=gpurun_out/dev
pf() {   # prefill throughput lines: prefill rows only, the mixed batch, the TP8 shard
  for a in "--no-decodes" "" "--tp 8"; do
    echo -n " [$a] $(env "$@" timeout 120 python scripts/bench_prefill.py --config llama70b $a 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'], 1))")"
  done
  echo
}
case "${1:-prefill}" in
  prefill)
    shift
    python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
    timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -3 | tee $O/prefill_tests.txt
    echo "default:$(pf X=1)" | tee $O/prefill_perf.txt
    for v in "$@"; do echo "$v:$(pf $v)" | tee -a $O/prefill_perf.txt; done ;;
  ab)
    shift
    python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
    echo "default:$(pf X=1)"
    for d in "$@"; do
      BKV_BUILD_DEFINES="$d" python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
      echo "$d:$(pf X=1)"
      timeout 300 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -1
    done
    python paper_2504_09590_b200/build.py --force > /dev/null 2>&1 ;;
  prefill-ncu)
    N=gpurun_out/dev_ncu; mkdir -p $N
    python paper_2504_09590_b200/build.py > /dev/null 2>&1
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 \
        -o $N/prefill python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes --steps 1 > $N/ncu.log 2>&1
    ncu -i $N/prefill.ncu-rep --page source --csv --print-source sass > $N/source_sass.csv 2> $N/src_err.txt
    ncu -i $N/prefill.ncu-rep --page raw --csv > $N/raw.csv 2>> $N/src_err.txt
    ls -la $N ;;
  decode)
    python paper_2504_09590_b200/build.py > /dev/null 2>&1
    timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fused_step.py tests/test_general_map_gpu.py tests/test_streams_graphs_gpu.py tests/test_reassembly_gpu.py -x -q 2>&1 | tail -3 | tee $O/dyn_tests.txt
    timeout 600 python scripts/quick_perf.py opt30b:1:fused llama70b:1:fused opt13b:1:fused llama70b:8:fused 2>&1 | tee $O/perf_dyn.txt ;;
esac

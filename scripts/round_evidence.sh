#!/bin/bash
# Round evidence on ONE GPU (run under gpurun; ~25 min).  Writes gpurun_out/r02/:
#   pytest_gpu.txt  smoke.txt  bench_*.json (opt13b default with shards, llama70b, opt30b,
#   general maps, reference arm)  sweep.jsonl (BASELINE configs[4], TP1/2/4/8)
#   prefill_*.json  sanitizer.txt  n2_gloo_smoke.txt, and the ncu captures (profile_r02.sh).
# ncu reports are summarised on the box into gpurun_out/r02_summary/ (copy to profiles/r02/ here).
set -u
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
step=${1:-all}
if [ $step = all ] || [ $step = tests ]; then
  timeout 3000 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -3 $O/smoke.txt
fi
if [ $step = all ] || [ $step = bench ]; then
  timeout 900 python bench.py > $O/bench_opt13b.json 2> $O/bench_err.txt
  timeout 900 python bench.py --config llama70b --no-shards > $O/bench_llama70b.json 2>> $O/bench_err.txt
  timeout 900 python bench.py --config opt30b --no-shards > $O/bench_opt30b.json 2>> $O/bench_err.txt
  timeout 900 python bench.py --general-map --no-shards --no-cpu > $O/bench_general_opt13b.json 2>> $O/bench_err.txt
  timeout 900 python bench.py --config llama70b --general-map --no-shards --no-cpu > $O/bench_general_llama70b.json 2>> $O/bench_err.txt
  timeout 600 python bench.py --impl reference > $O/bench_ref.json 2>> $O/bench_err.txt
  bash scripts/n2_smoke.sh > $O/n2_gloo_smoke.txt 2>&1
fi
if [ $step = all ] || [ $step = sweep ]; then
  timeout 1500 python scripts/sweep_bench.py --L0 512 2048 8192 --rt 1 0.5 0 > $O/sweep.jsonl 2>> $O/sweep_err.txt
fi
if [ $step = all ] || [ $step = prefill ]; then
  timeout 900 python scripts/bench_prefill.py --config llama70b --tp 1 > $O/prefill_llama70b_tp1.json 2>> $O/prefill_err.txt
  timeout 900 python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes > $O/prefill_llama70b_tp1_prefill_only.json 2>> $O/prefill_err.txt
  timeout 900 python scripts/bench_prefill.py --config llama70b --tp 8 > $O/prefill_llama70b_tp8.json 2>> $O/prefill_err.txt
  # ncu of the prefill kernel alone; key metrics extracted on the box -> prefill_ncu.txt
  timeout 600 ncu --set full --clock-control none -k regex:prefill_tc -s 2 -c 1 -o $O/prefill_ncu \
      python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes --steps 1 > $O/prefill_ncu.log 2>&1
  ncu -i $O/prefill_ncu.ncu-rep --page raw --csv > $O/prefill_raw.csv 2>> $O/prefill_err.txt && \
      python scripts/ncu_prefill_metrics.py $O/prefill_raw.csv > $O/prefill_ncu.txt 2>> $O/prefill_err.txt
  rm -f $O/prefill_ncu.ncu-rep $O/prefill_raw.csv
fi
if [ $step = all ] || [ $step = sanitize ]; then
  for tool in memcheck racecheck initcheck synccheck; do
    echo "== $tool" >> $O/sanitizer.txt
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_target.py >> $O/sanitizer.txt 2>&1
    echo "exit $?" >> $O/sanitizer.txt
  done
fi
if [ $step = all ] || [ $step = ncu ]; then
  timeout 2400 bash scripts/profile_r02.sh > $O/profile.log 2>&1
  # summarise on the box (gpurun copies back <= 64 MiB): the .ncu-rep files stay there
  mkdir -p gpurun_out/r02_summary
  BKV_SUMMARY_DST=gpurun_out/r02_summary python scripts/summarize_r02.py > $O/summarize.log 2>&1
  rm -f gpurun_out/prof_r02/*.ncu-rep
fi
ls -la $O

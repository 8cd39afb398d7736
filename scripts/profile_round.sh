#!/bin/bash
# Capture the round's ncu evidence on ONE GPU (run under gpurun):
#  1. launch lists (device time of every kernel) of short bench.py runs (opt13b, llama70b)
#  2. --set full captures of the decode kernel on the bench config and the TP shard shapes
#  3. full captures of the merge, append, prefill kernels
# Output: gpurun_out/prof_<round>/  (summarise with scripts/summarize_profiles.py <round>)
set -u
R=${1:-r01}
OUT=gpurun_out/prof_$R
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_opt13b.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $OUT/launches_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_llama70b.csv \
    python bench.py --config llama70b --layers 8 --steps 2 --warmup 3 --no-cpu > $OUT/launches_bench_llama.log 2>&1
for c in "opt13b 1" "opt13b 2" "opt30b 4" "llama70b 8" "llama70b 4" "llama70b 1"; do
  set -- $c
  ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 6 -c 1 \
      -o $OUT/decode_$1_tp$2 python scripts/ncu_target.py $1 $2 8 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:merge_kernel -s 6 -c 1 \
    -o $OUT/merge_llama70b_tp1 python scripts/ncu_target.py llama70b 1 8 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:kv_append -s 6 -c 1 -o $OUT/append_opt13b_tp1 \
    python scripts/ncu_target.py opt13b 1 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefill -s 2 -c 1 \
    -o $OUT/prefill_llama70b_tp1 python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes --steps 1 > /dev/null 2>&1
ls -la $OUT

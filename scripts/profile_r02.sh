#!/bin/bash
# Round r02 ncu evidence on ONE GPU (run under gpurun):
#  1. launch lists (device time of every kernel) of short bench.py runs (opt13b, llama70b)
#  2. --set full captures of the planned decode (decode + cross-CTA merge kernels) of every shard,
#     three layers (six launches) each: SURVEY §8(d) asks for >= 3 launches per config
#  3. the dynamic kernel pair of the large OPT-30B TP1 problem, the append and prefill kernels
# Output: gpurun_out/prof_r02/ (summarise with scripts/summarize_r02.py)
set -u
OUT=gpurun_out/prof_r02
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_opt13b.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-shards > $OUT/launches_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_llama70b.csv \
    python bench.py --config llama70b --layers 8 --steps 2 --warmup 3 --no-cpu --no-shards > $OUT/launches_bench_llama.log 2>&1
for c in "llama70b 1" "llama70b 2" "llama70b 4" "llama70b 8" "opt13b 1" "opt13b 2" "opt13b 4" "opt13b 8" "opt30b 4"; do
  set -- $c
  ncu --set full --clock-control none --import-source on -k regex:planned -s 12 -c 6 \
      -o $OUT/planned_$1_tp$2 python scripts/ncu_target_planned.py $1 $2 12 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|merge_kernel" -s 8 -c 6 \
    -o $OUT/dynamic_opt30b_tp1 python scripts/ncu_target_planned.py opt30b 1 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefill -s 2 -c 1 \
    -o $OUT/prefill_llama70b_tp1 python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes --steps 1 > /dev/null 2>&1
ls -la $OUT

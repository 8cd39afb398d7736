# dev: launch-parameter sweep of the decode kernel on the small (TP8-shard) shapes
set -u
OUT=gpurun_out/sweep_${1:-a}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in llama70b:8:fused opt13b:8:fused opt13b:2:fused llama70b:1:fused; do
 for S in 2 3; do
  for MS in 4 8 16; do
   for UPW in 1 3; do
    BKV_SLOTS=$S BKV_MIN_SPLIT=$MS BKV_UNITS_PER_WARP=$UPW timeout 120 python scripts/quick_perf.py $cfg 2>&1 | tail -n1 | sed "s/^/S=$S MS=$MS UPW=$UPW /" >> $OUT/sweep.txt
   done
  done
 done
done

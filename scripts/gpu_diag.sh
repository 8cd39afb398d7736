# dev: GPU tests + small-shape diagnosis (trace timeline, data-movement skeleton)
set -u
OUT=gpurun_out/diag_${1:-a}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest $?" >> $OUT/status
for c in llama70b:8 opt13b:8 opt13b:1; do
  IFS=: read cfg tp <<< "$c"
  timeout 120 python scripts/trace_run.py $cfg $tp >> $OUT/trace.txt 2>&1
  BKV_DEBUG=1 timeout 120 python scripts/quick_perf.py $cfg:$tp >> $OUT/skeleton.txt 2>&1
  timeout 120 python scripts/quick_perf.py $cfg:$tp >> $OUT/skeleton.txt 2>&1
done

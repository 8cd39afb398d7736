# dev: GPU tests + A/B of an env switch on the per-layer timing (quick_perf)
# usage: bash scripts/gpu_ab.sh TAG VAR "v0 v1" "cfg:tp[:mode] ..."
set -u
OUT=gpurun_out/ab_$1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest $?" >> $OUT/status
for spec in $4; do
  for v in $3; do
    env $2=$v timeout 120 python scripts/quick_perf.py $spec 2>&1 | tail -n1 | sed "s/^/$2=$v /" >> $OUT/ab.txt
  done
done

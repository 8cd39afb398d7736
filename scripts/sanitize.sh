# compute-sanitizer on scripts/sanitize_target.py (run under gpurun; one GPU)
set -u
OUT=gpurun_out/sanitize_${1:-a}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for tool in memcheck racecheck initcheck synccheck; do
  echo "== $tool" >> $OUT/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_target.py >> $OUT/sanitizer.txt 2>&1
  echo "exit $?" >> $OUT/sanitizer.txt
done

set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1
true
BKV_BUILD_TRACE=1 python paper_2504_09590_b200/build.py --force > /dev/null 2>&1
for s in "llama70b 8 6 early"; do BKV_TRACE=8 timeout 300 python scripts/trace_planned.py $s; done 2>&1 | tee gpurun_out/trace_planned.txt
python paper_2504_09590_b200/build.py --force > /dev/null 2>&1

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1
timeout 2400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/x_tests.txt
bash scripts/round_evidence.sh sanitize
bash scripts/round_evidence.sh sweep

cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 1 > $O/prefill_llama70b_tp1.json 2>> $O/prefill_err.txt
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes > $O/prefill_llama70b_tp1_prefill_only.json 2>> $O/prefill_err.txt
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 8 > $O/prefill_llama70b_tp8.json 2>> $O/prefill_err.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill -s 2 -c 1 \
    -o $O/prefill_llama70b_tp1 python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes --steps 1 > $O/ncu.log 2>&1
ncu -i $O/prefill_llama70b_tp1.ncu-rep --page raw --csv > $O/prefill_raw.csv 2>&1
rm -f $O/*.ncu-rep
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_fused_step.py -q > $O/pytest_prefill.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
ls -la $O

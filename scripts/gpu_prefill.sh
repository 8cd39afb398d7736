# dev: prefill measurement + ncu capture (run under gpurun)
set -u
OUT=gpurun_out/prefill_${1:-a}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 1 > $OUT/bench_llama_tp1.json 2> $OUT/err1.log
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 8 > $OUT/bench_llama_tp8.json 2> $OUT/err2.log
timeout 300 python scripts/bench_prefill.py --config opt13b --tp 2 > $OUT/bench_opt13b_tp2.json 2> $OUT/err3.log
timeout 600 python scripts/bench_prefill.py --config llama70b --tp 8 --steps 5 --cost-model $OUT/cost_model_llama70b_tp8.csv > $OUT/cost_fit.json 2> $OUT/err4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 4 -c 1 \
    -o $OUT/prefill_llama_tp1 python scripts/bench_prefill.py --config llama70b --tp 1 --steps 1 > $OUT/ncu.log 2>&1

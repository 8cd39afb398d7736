# round evidence: tests, smoke, bench lines (3 configs + oracle reference arm), N=2 smoke of the multi-GPU path
set -u
R=${1:-r01e}
OUT=gpurun_out/final_$R
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest $?" >> $OUT/status
timeout 600 python bench.py > $OUT/bench_opt13b.json 2> $OUT/bench_opt13b.err; echo "bench opt13b $?" >> $OUT/status
for c in llama70b opt30b; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c $?" >> $OUT/status
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref $?" >> $OUT/status
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 1 > $OUT/bench_prefill_llama_tp1.json 2>&1
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 8 > $OUT/bench_prefill_llama_tp8.json 2>&1
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes > $OUT/bench_prefill_llama_tp1_prefill_only.json 2>&1
timeout 300 python scripts/bench_prefill.py --config opt13b --tp 2 > $OUT/bench_prefill_opt13b_tp2.json 2>&1
timeout 600 python scripts/sweep_bench.py > $OUT/sweep_llama70b.jsonl 2> $OUT/sweep.err; echo "sweep $?" >> $OUT/status
timeout 300 python scripts/quick_perf.py llama70b:1:fused llama70b:2:fused llama70b:4:fused llama70b:8:fused opt13b:1:fused opt13b:2:fused opt13b:4:fused opt13b:8:fused opt30b:1:fused opt30b:4:fused > $OUT/quick_perf.txt 2>&1
timeout 600 python scripts/bench_prefill.py --config llama70b --tp 8 --steps 5 --cost-model $OUT/cost_model_llama70b_tp8.csv > $OUT/cost_fit.json 2>&1
BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --layers 4 --no-cpu > $OUT/n2_gather.log 2>&1; echo "n2 gather $?" >> $OUT/status
BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 3 --warmup 3 --layers 4 --no-cpu --reassembly p2p > $OUT/n2_p2p.log 2>&1; echo "n2 p2p $?" >> $OUT/status

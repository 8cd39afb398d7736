python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r9
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r9/pytest.log 2>&1
timeout 300 python scripts/bench_prefill.py --config llama70b --tp 1 > gpurun_out/r9/bench_prefill_llama_tp1.json 2>&1
BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config opt13b --steps 3 --warmup 3 --layers 4 --reassembly p2p > gpurun_out/r9/p2p_gloo2.log 2>&1; echo "p2p exit $?" >> gpurun_out/r9/p2p_gloo2.log
BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config opt13b --steps 3 --warmup 3 --layers 4 > gpurun_out/r9/nccl_gloo2.log 2>&1; echo "gather exit $?" >> gpurun_out/r9/nccl_gloo2.log

python -c "import __graft_entry__ as g; g.build()" > /dev/null
mkdir -p gpurun_out/r10
timeout 600 python -m pytest tests/test_reassembly_mp_gpu.py tests/test_reassembly_gpu.py -x -q > gpurun_out/r10/pytest_re.log 2>&1
BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config opt13b --steps 3 --warmup 3 --layers 4 --reassembly p2p --no-cpu > gpurun_out/r10/p2p_gloo2.log 2>&1; echo "p2p exit $?" >> gpurun_out/r10/p2p_gloo2.log
BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config opt13b --steps 3 --warmup 3 --layers 4 --no-cpu > gpurun_out/r10/nccl_gloo2.log 2>&1; echo "gather exit $?" >> gpurun_out/r10/nccl_gloo2.log
for c in llama70b:8:fused opt13b:8:fused opt13b:1:fused llama70b:1:fused; do timeout 120 python scripts/quick_perf.py $c >> gpurun_out/r10/perf.txt 2>&1; done

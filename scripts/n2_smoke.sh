# N=2 smoke of bench.py's multi-GPU path on ONE GPU (gloo backend, 2 ranks): per-step and per-layer gather, p2p
for extra in "" "--gather layer" "--reassembly p2p"; do
  BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 --layers 4 --no-cpu $extra 2>gpurun_out/n2_err.txt | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$extra', d['value'], d['detail']['reassembly'], d['detail']['reassembly_ms_per_step'], d['e2e'])" || tail -20 gpurun_out/n2_err.txt
done

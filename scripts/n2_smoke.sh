# N=2 smoke of bench.py's multi-GPU path on ONE GPU (gloo backend, 2 ranks): per-step and per-layer gather, p2p
for extra in "" "--gather layer" "--reassembly p2p"; do
  BKV_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 --layers 4 --no-cpu $extra 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$extra', d['value'], d['config']['reassembly'], d['e2e'])"
done

set -u
mkdir -p gpurun_out/r01c
cp MEASURED_PEAKS.json gpurun_out/r01c/ 2>/dev/null; ls /root/repo/ > gpurun_out/r01c/ls.txt
nvidia-smi > gpurun_out/r01c/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r01c/smoke.log 2>&1; echo smoke $? >> gpurun_out/r01c/status
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r01c/pytest_gpu.log 2>&1; echo pytest $? >> gpurun_out/r01c/status
for c in opt13b llama70b opt30b; do
  timeout 600 python bench.py --config $c > gpurun_out/r01c/bench_$c.json 2> gpurun_out/r01c/bench_$c.err; echo bench $c $? >> gpurun_out/r01c/status
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01c/bench_ref.json 2> gpurun_out/r01c/bench_ref.err
timeout 1500 bash scripts/profile_round.sh r01c > gpurun_out/r01c/prof.log 2>&1; echo prof $? >> gpurun_out/r01c/status

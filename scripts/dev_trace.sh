#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out/dev
python paper_2504_09590_b200/build.py > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fused_step.py tests/test_general_map_gpu.py tests/test_streams_graphs_gpu.py tests/test_reassembly_gpu.py -x -q 2>&1 | tail -3 | tee gpurun_out/dev/dyn_tests.txt
timeout 600 python scripts/quick_perf.py opt30b:1:fused llama70b:1:fused opt13b:1:fused llama70b:8:fused 2>&1 | tee gpurun_out/dev/perf_dyn.txt

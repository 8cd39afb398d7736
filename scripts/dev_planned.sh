set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_2504_09590_b200/build.py > /dev/null 2>&1 || python paper_2504_09590_b200/build.py
timeout 600 python scripts/quick_perf.py llama70b:8:planned_early llama70b:4:planned_early llama70b:2:planned_early llama70b:1:planned_early opt13b:8:planned_early opt13b:4:planned_early opt13b:2:planned_early opt13b:1:planned_early opt30b:4:planned_early 2>&1 | tee gpurun_out/planned_perf.txt
ncu --set full --clock-control none -k regex:planned -s 12 -c 2 -o gpurun_out/prof_tp8 python scripts/ncu_target_planned.py llama70b 8 8 > /dev/null 2>&1
ncu -i gpurun_out/prof_tp8.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum 2>&1 | tail -3 > gpurun_out/prof_tp8.txt
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 | tee gpurun_out/gpu_tests.txt

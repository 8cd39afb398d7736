set -u
R=${1:-r01f}
bash scripts/gpu_final.sh $R
bash scripts/sanitize.sh $R
bash scripts/profile_round.sh $R > gpurun_out/prof_$R.log 2>&1

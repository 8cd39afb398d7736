# dev: A/B of the mixed dispatch overlap (decode part alongside the prefill tail)
for ov in 1 0 1 0; do
  echo "overlap $ov"
  BKV_MIXED_OVERLAP=$ov python scripts/bench_prefill.py --config llama70b --tp 1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('llama tp1', round(d['value'],1), d['us_per_layer'])"
  BKV_MIXED_OVERLAP=$ov python scripts/bench_prefill.py --config llama70b --tp 8 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('llama tp8', round(d['value'],1), d['us_per_layer'])"
  BKV_MIXED_OVERLAP=$ov python scripts/bench_prefill.py --config opt13b --tp 2 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('opt13b tp2', round(d['value'],1), d['us_per_layer'])"
done

python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('llama tp1 prefill-only', round(d['value'],1), d['us_per_layer'])"
python scripts/bench_prefill.py --config llama70b --tp 1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('llama tp1 mixed', round(d['value'],1), d['us_per_layer'])"
python scripts/bench_prefill.py --config llama70b --tp 8 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('llama tp8 mixed', round(d['value'],1), d['us_per_layer'])"
python scripts/bench_prefill.py --config opt13b --tp 2 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('opt13b tp2 mixed', round(d['value'],1), d['us_per_layer'])"

# full GPU suite + headline and config-4b timing
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['encode_ms'], d['decode_ms'])"
timeout 300 python bench.py --workload pcw --no-cpu --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pcw', d['value'], d['ms_per_step'])"

# parity + headline timing
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in 0 0 0; do
  timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['encode_ms'], d['decode_ms'])"
done

# row-only raw instances A/B (LCH_NO_ROWONLY=1 keeps the packet-capable ones) + parity
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in 0 1 0 1 0 1; do
  if [ $v = 1 ]; then export LCH_NO_ROWONLY=1; else unset LCH_NO_ROWONLY; fi
  timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_rowonly=$v', d['value'], d['encode_ms'], d['decode_ms'])"
done

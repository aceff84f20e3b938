# inverse-pattern lean instance A/B (LCH_NO_INVPAT2=1 keeps the shaped instance)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for v in 0 1 0 1 0 1; do
  if [ $v = 1 ]; then export LCH_NO_INVPAT2=1; else unset LCH_NO_INVPAT2; fi
  timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_invpat2=$v', d['value'], d['encode_ms'], d['decode_ms'])"
done

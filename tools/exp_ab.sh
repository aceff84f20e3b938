# parity + headline timing + per-launch durations of the headline step
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in 0 0; do
  timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['encode_ms'], d['decode_ms'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pass_kernel|gather" --csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 2>/dev/null | grep gpu__time | awk -F'","' '{printf "%s ", $NF} END {print ""}'

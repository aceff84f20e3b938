# parity + A/B timing of the two pass pipelines (LCH_PASS_TEAMS=1 single-team)
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -x -q -m gpu 2>&1 | tail -3
for t in 2 1 2; do LCH_PASS_TEAMS=$t timeout 120 python tools/time_encode.py | sed "s/^/teams=$t /"; done
for t in 2 1; do LCH_PASS_TEAMS=$t timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('teams=$t bench', d['value'], d['encode_ms'], d['decode_ms'])"; done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel -s 10 -c 5 --csv python tools/time_encode.py 2>/dev/null | grep gpu__time | awk -F'","' '{printf "%s ", $NF} END {print ""}'

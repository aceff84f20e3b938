# parity + config-4b timing + per-launch durations of the per-codeword decode
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python bench.py --workload pcw --no-cpu --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pcw', d['value'], d['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"locator16|pass_kernel|gather" --csv python bench.py --workload pcw --no-cpu --steps 1 --warmup 0 2>/dev/null | grep gpu__time | awk -F'","' '{printf "%s ", $NF} END {print ""}'

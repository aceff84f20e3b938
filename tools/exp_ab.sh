# parity + headline timing + gather launch durations
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['encode_ms'], d['decode_ms'])"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gather" -c 2 --csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 --only decode 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{printf "%s %s | ", $(NF-2), $NF} END {print ""}'

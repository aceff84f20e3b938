# A/B of alternative builds (LCH_SO_PATH): headline step + gather launch time
for so in paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_*/liblch.so paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_*/liblch.so; do
  LCH_SO_PATH=$so timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', d['value'], d['encode_ms'], d['decode_ms'])"
done
for so in paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_*/liblch.so; do
LCH_SO_PATH=$so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gather" -c 2 --csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 1 --only decode 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{printf "%s %s | ", $(NF-2), $NF} END {print ""}'
done
LCH_SO_PATH=paper_1404_3458_b200/_build_g3/liblch.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stripe.py -x -q -m gpu 2>&1 | tail -2

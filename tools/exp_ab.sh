# A/B of alternative builds (LCH_SO_PATH): headline step encode/decode
for so in paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_*/liblch.so paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_*/liblch.so; do
  LCH_SO_PATH=$so timeout 200 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', d['value'], d['encode_ms'], d['decode_ms'])"
done

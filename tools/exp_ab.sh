# A/B encode + decode timing of alternative builds (LCH_SO_PATH) and a parity check
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for so in paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_*/liblch.so; do
  for i in 1 2; do
    LCH_SO_PATH=$so python tools/time_encode.py | sed "s|^|$so |"
  done
done
python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['encode_ms'], d['decode_ms'])"
LCH_SO_PATH=paper_1404_3458_b200/_build_1bit/liblch.so python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench1bit', d['value'], d['encode_ms'], d['decode_ms'])"

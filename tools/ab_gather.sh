# headline step and gather kernel time for (LCH_GATHER_DIRECT, LCH_GATHER_LW) pairs
for cfg in "0 1" "3 4" "3 3" "2 2" "4 4" "3 2" "4 3" "2 3"; do
  set -- $cfg
  export LCH_GATHER_DIRECT=$1 LCH_GATHER_LW=$2
  timeout 200 python bench.py --no-cpu --no-e2e --no-aux --steps 10 --warmup 3 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct=$1 lw=$2', d['value'], d['encode_ms'], d['decode_ms'])"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gather -s 3 -c 1 python tools/time_codec.py 2>&1 | grep -E "gather_kernel|gpu__time|dram__bytes"
done

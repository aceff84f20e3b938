# A/B of one environment knob on the headline step: bash tools/ab_env.sh VAR [reps]
# (prints value / encode ms / decode ms with the knob unset and set, interleaved)
VAR=$1; REPS=${2:-3}
for i in $(seq $REPS); do
  for on in 0 1; do
    if [ $on = 1 ]; then export $VAR=1; else unset $VAR; fi
    timeout 200 python bench.py --no-cpu --no-e2e --no-aux --steps 10 --warmup 3 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$on', d['value'], d['encode_ms'], d['decode_ms'])"
  done
done
unset $VAR

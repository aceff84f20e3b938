# Round profile captures (each command exits 0 without ncu first):
#  1. launch list of the headline bench step (encode 4096 + shared-pattern decode 4096)
#  2. --set full of two encode pass_kernel launches (BS->BS pass and the fused 10-level pass)
#  (the LCH_DBG_PASS bisection, tools/exp_passes.sh, needs a -DLCH_PASS_DBG build)
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_bench.json 2>gpurun_out/prof_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s 6 -c 2 \
  -o gpurun_out/pass_full python tools/time_encode.py > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel -s 10 -c 5 --csv python tools/time_encode.py > gpurun_out/encode_passes.csv 2>/dev/null

# Round profile captures (each command exits 0 without ncu first):
#  1. launch list of tools/time_codec.py (headline encode + shared-pattern decode, 4096 codewords)
#  2. --set full of one encode (5 pass launches) and one decode (6 passes + gather), with SASS source
#  (the LCH_DBG_PASS bisection, tools/exp_passes2.sh, needs a -DLCH_PASS_DBG build)
set -x
TAG=${TAG:-r02b}
python tools/time_codec.py > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
if [ -z "$SKIP_LAUNCHES" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python tools/time_codec.py > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/ncu_summary.py launches gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_launches.md
fi
ncu --set full --import-source on --clock-control none -k regex:"pass_kernel|gather" -s 13 -c 5 \
  -f -o gpurun_out/${TAG}_encode python tools/time_codec.py > gpurun_out/${TAG}_ncu_enc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"pass_kernel|gather" -s 78 -c 7 \
  -f -o gpurun_out/${TAG}_decode python tools/time_codec.py > gpurun_out/${TAG}_ncu_dec.log 2>&1
# summaries made on the box (the reports are too big to travel back)
python tools/ncu_summary.py full gpurun_out/${TAG}_encode.ncu-rep gpurun_out/${TAG}_encode_passes_full.txt gpurun_out/${TAG}_traffic.json
python tools/ncu_summary.py full gpurun_out/${TAG}_decode.ncu-rep gpurun_out/${TAG}_decode_kernels_full.txt
: > gpurun_out/${TAG}_opcode_profiles.md
for w in encode decode; do
  ncu -i gpurun_out/${TAG}_$w.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_${w}_src.csv 2>/dev/null
  n=5; [ $w = decode ] && n=7
  for i in $(seq 0 $((n - 1))); do
    echo "## ${TAG}_$w launch $i" >> gpurun_out/${TAG}_opcode_profiles.md
    echo '```' >> gpurun_out/${TAG}_opcode_profiles.md
    python tools/sass_profile.py /tmp/${TAG}_${w}_src.csv $i >> gpurun_out/${TAG}_opcode_profiles.md 2>&1
    echo '```' >> gpurun_out/${TAG}_opcode_profiles.md
  done
done
rm -f gpurun_out/${TAG}_encode.ncu-rep gpurun_out/${TAG}_decode.ncu-rep

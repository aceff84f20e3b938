export LCH_SO_PATH=$PWD/paper_1404_3458_b200/_build_dbg/liblch.so
for d in 0 1 2 3 32 34 64 33 35; do
  LCH_DBG_PASS=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel -s 10 -c 5 --csv python tools/time_encode.py 2>/dev/null | grep gpu__time | awk -F'","' -v d=$d '{printf "%s ", $NF} END {print " dbg=" d}'
done

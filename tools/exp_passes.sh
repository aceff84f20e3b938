# per-launch durations (ns) of the 5 encode passes under LCH_DBG_PASS bisection
# (library built with: make -C paper_1404_3458_b200/csrc EXTRA=-DLCH_PASS_DBG)
# flags: 0 normal, 1 no global I/O, 2 no butterflies, 3 neither (results wrong when set)
for d in 0 1 2 3; do
  LCH_DBG_PASS=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pass_kernel -s 10 -c 5 --csv python tools/time_encode.py 2>/dev/null | grep gpu__time | awk -F'","' -v d=$d '{printf "%s ", $NF} END {print " dbg=" d}'
done

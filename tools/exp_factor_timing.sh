# encode timing under LCH_DBG_PASS bisection flags (results wrong when set)
for d in 0 2 3 34 130 66 1 32 128 64 0x80000100 0x80000102; do
  LCH_DBG_PASS=$d python tools/time_encode.py
done

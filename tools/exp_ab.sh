# host compaction A/B: streaming-store compaction (_build) vs compress-store (_build_old)
timeout 600 python -m pytest tests/test_gpu_host.py -x -q -m gpu 2>&1 | tail -2
for rep in 1 2 3; do
for so in paper_1404_3458_b200/_build/liblch.so paper_1404_3458_b200/_build_old/liblch.so; do
  echo "$so $(LCH_SO_PATH=$so timeout 120 python tools/compact_bw.py 4096 2>&1 | tail -1) | $(LCH_SO_PATH=$so timeout 300 python tools/e2e_phases.py 2>&1 | grep -E 'decode_host:|both' | tr '\n' ' ')"
done
done

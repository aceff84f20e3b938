# round-end style check: GPU tests, smoke, and every bench line (1 GPU)
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
bash tools/all_workloads.sh

# round-end style check: GPU tests, smoke, every bench line (1 GPU), and a
# 2-rank torchrun run on the one GPU through the gloo barrier
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
bash tools/all_workloads.sh
LCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/wl_2rank.json 2> gpurun_out/wl_2rank.err

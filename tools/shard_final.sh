timeout 600 python tools/shard_time.py --config 4 --gpus 1 2 4 8 --steps 2 > gpurun_out/shard_final.log 2>&1
timeout 400 python tools/shard_time.py --config 4 --gpus 1 2 4 8 --steps 2 --factorization ldlt >> gpurun_out/shard_final.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests6.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke6.log 2>&1

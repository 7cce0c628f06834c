for cfg in 2 4; do timeout 300 python tools/laswp_ab.py $cfg >> gpurun_out/ab2.log 2>&1; done
timeout 900 python -m pytest -q -x tests -m gpu > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests2.log
bash tools/stream_ncu.sh

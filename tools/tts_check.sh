timeout 400 python tools/tts_phases.py 4 > gpurun_out/tts_phases2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests4.log
timeout 900 python bench.py > gpurun_out/bench4.log 2>&1; echo "bench rc=$?"

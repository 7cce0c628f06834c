timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests5.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests5.log
timeout 400 python tools/tts_phases.py 3 > gpurun_out/tts_phases3.log 2>&1
timeout 400 python tools/tts_phases.py 0 > gpurun_out/tts_phases0.log 2>&1

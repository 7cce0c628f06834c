# closing batch: GPU tests, bench line, outer-block A/B at cfg2 / cfg3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests3.log
timeout 900 python bench.py > gpurun_out/bench3.log 2>&1; echo "bench rc=$?"
for cfg in 2 3; do for lp in 4 8 16; do
  echo -n "LU_PANELS=$lp " >> gpurun_out/abmid.log
  FEASTLAB_LU_PANELS=$lp timeout 300 python tools/laswp_ab.py $cfg >> gpurun_out/abmid.log 2>&1
done; done

# LU outer-block width A/B at cfg4 (application ms) and its parity tests
for lp in 8 12 16; do
  echo -n "LU_PANELS=$lp " >> gpurun_out/ab16.log
  FEASTLAB_LU_PANELS=$lp timeout 300 python tools/laswp_ab.py 4 >> gpurun_out/ab16.log 2>&1
done
for lp in 8 16; do
  echo -n "LDLT LU_PANELS=$lp " >> gpurun_out/ab16.log
  FEASTLAB_FACTOR=ldlt FEASTLAB_LU_PANELS=$lp timeout 300 python tools/laswp_ab.py 4 >> gpurun_out/ab16.log 2>&1
done
timeout 600 python -m pytest -q -x tests/test_gpu_blocks.py tests/test_gpu_ldlt.py >> gpurun_out/ab16.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab16.log

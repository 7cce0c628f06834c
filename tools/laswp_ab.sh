# laswp A/B: bitwise Y digests and application time for both forms, plus the
# laswp launch durations under ncu (cfg2), then the GPU LU tests on the new form
for cfg in 2 3 4; do
  for m in smem warp; do
    FEASTLAB_LASWP=$m timeout 300 python tools/laswp_ab.py $cfg >> gpurun_out/laswp_ab.log 2>&1
  done
done
for m in smem warp; do
  FEASTLAB_LASWP=$m timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:laswp -c 200 --csv --log-file gpurun_out/laswp_ncu_$m.csv python tools/laswp_ab.py 2 > /dev/null 2>&1
done
timeout 900 python -m pytest -q -x tests/test_gpu_blocks.py tests/test_gpu_exact.py tests/test_gpu_configs.py > gpurun_out/laswp_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/laswp_tests.log

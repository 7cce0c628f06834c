# correctness + timing of the LU / solve block widths (FEASTLAB_LU_PANELS, FEASTLAB_SOLVE_PANELS)
for lp in "2 2" "4 4" "3 3" "4 2" "2 4"; do
  set -- $lp
  echo "LU=$1 SOLVE=$2" >> gpurun_out/ab.log
  FEASTLAB_LU_PANELS=$1 FEASTLAB_SOLVE_PANELS=$2 timeout 300 python -m pytest -q -x tests/test_gpu_configs.py -k "first_filtered or cfg0" tests/test_gpu_exact.py -k "first_filtered or cfg0 or cfg3" 2>&1 | tail -2 >> gpurun_out/ab.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for cfg in "2 1" "2 8" "2 4"; do
 for lp in "2 2" "4 4" "2 4"; do
  set -- $lp
  echo -n "LU=$1 SOLVE=$2 " >> gpurun_out/ab.log
  FEASTLAB_LU_PANELS=$1 FEASTLAB_SOLVE_PANELS=$2 timeout 200 python tools/shard_floor.py $cfg >> gpurun_out/ab.log 2>&1
 done
done

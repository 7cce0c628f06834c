for lp in 16 32; do
  echo -n "LU_PANELS=$lp " >> gpurun_out/ab32.log
  FEASTLAB_LU_PANELS=$lp timeout 300 python tools/laswp_ab.py 4 >> gpurun_out/ab32.log 2>&1
done
timeout 300 python tools/tts_phases.py 4 > gpurun_out/tts_phases.log 2>&1

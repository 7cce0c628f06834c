# one ncu --set full capture of the TMA-fed trailing updates at cfg4 (16-panel outer
# blocks: K = 1024 trailing updates); the report is read back here
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:zgemm3s --launch-skip 24 --launch-count 2 -o gpurun_out/zgemm3s_cfg4 -f python tools/one_app.py 4 lu 1 > gpurun_out/zgemm_full.log 2>&1; echo "ncu rc=$?"

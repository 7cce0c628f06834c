# one ncu --set full capture of zgemm3m launches at cfg4 (16-panel outer
# blocks: K = 1024 trailing updates); the report is read back here
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:zgemm3m_kernel --launch-skip 100 --launch-count 40 -o gpurun_out/zgemm3m_k1024 python tools/filter_once.py 4 1 > gpurun_out/zgemm_full.log 2>&1; echo "ncu rc=$?"

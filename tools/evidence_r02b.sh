set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r02b.txt 2>&1; tail -3 gpurun_out/gpu_tests_r02b.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.txt 2>&1; tail -1 gpurun_out/smoke_r02b.txt
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:zgemm|laswp|compose_perm' --csv --log-file gpurun_out/zt.csv python tools/one_app.py 4 lu 1 > gpurun_out/zt.log 2>&1; echo "traffic rc=$?"
python tools/zgemm_traffic.py gpurun_out/zt.csv 4 > gpurun_out/ncu_zgemm_traffic_cfg4_r02b.json && gzip -f gpurun_out/zt.csv
timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_r02b.csv python bench.py --steps 1 --warmup 3 --no-tts --no-cpu-baseline --no-alt --streams 1 > gpurun_out/launches_ncu.log 2>&1; echo "launch list rc=$?"
python tools/ncu_summary.py gpurun_out/launches_cfg4_r02b.csv > gpurun_out/launches_cfg4_r02b.json && gzip -f gpurun_out/launches_cfg4_r02b.csv
ls -la gpurun_out | tail -8

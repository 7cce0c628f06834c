# round-1 closing measurements: bench line, the cfg4 launch list of one
# application, HBM counters of accumulate / permute_rhs
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_final.csv python tools/one_app.py 4 > gpurun_out/launches_final.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k 'regex:accumulate_kernel|permute_rhs|shift_kernel' --csv --log-file gpurun_out/stream_acc_cfg4.csv python tools/one_app.py 4 > gpurun_out/stream_acc.log 2>&1; echo "acc rc=$?"

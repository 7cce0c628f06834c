# ncu HBM counters of the streaming kernels: the filter's (shift, laswp,
# permute_rhs, accumulate) on one cfg4 application and the Rayleigh-Ritz
# tail's (column norms, residual, scaling, gathers, symmetrisation) on a cfg2
# FEAST solve. Output: gpurun_out/stream_*.csv
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k 'regex:shift_kernel|accumulate_kernel|permute_rhs|laswp' -c 1200 --csv --log-file gpurun_out/stream_filter_cfg4.csv python tools/one_app.py 4 > gpurun_out/stream_filter.log 2>&1; echo "filter ncu rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k 'regex:col_norms|residual_kernel|col_div|gather_cols|symmetrize|transpose_kernel|tril_kernel' -c 400 --csv --log-file gpurun_out/stream_rr_cfg2.csv python tools/rr_once.py 2 > gpurun_out/stream_rr.log 2>&1; echo "rr ncu rc=$?"

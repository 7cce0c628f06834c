# reference arm (driver-like and short), GEMM shape classes of the final build, ncu --set full of one composed interchange pass
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_cfg4_r02.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_cfg4_r02_k20.json 2>> gpurun_out/bench_ref.err; echo "ref k20 rc=$?"
python tools/zgemm_classes.py 4 1 > gpurun_out/zgemm_classes_cfg4_serial_r02.json 2> gpurun_out/zc1.err; echo "classes serial rc=$?"
python tools/zgemm_classes.py 4 8 > gpurun_out/zgemm_classes_cfg4_8streams_r02.json 2> gpurun_out/zc8.err; echo "classes 8 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:laswp_block --launch-skip 6 --launch-count 1 -o gpurun_out/laswp_block_cfg4_r02 -f python tools/one_app.py 4 lu 1 > gpurun_out/laswp_full.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/*.ncu-rep | tail -3

for lp in 1 2 4; do
  echo "LU_PANELS=$lp" >> gpurun_out/shard_cfg2.log
  FEASTLAB_LU_PANELS=$lp timeout 300 python tools/shard_time.py --config 2 --gpus 8 4 2 --steps 5 >> gpurun_out/shard_cfg2.log 2>&1
done
echo "default" >> gpurun_out/shard_cfg2.log
timeout 300 python tools/shard_time.py --config 2 --gpus 1 2 4 8 --steps 5 >> gpurun_out/shard_cfg2.log 2>&1
timeout 300 python tools/shard_time.py --config 2 --gpus 1 2 4 8 --steps 5 --factorization ldlt >> gpurun_out/shard_cfg2.log 2>&1

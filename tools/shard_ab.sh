# cfg4 shard time per outer-block width at 2/4/8 GPUs (4..16 local nodes),
# then the default strong-scaling table (LU and LDL^T)
for lp in 2 4 8 16; do
  echo "LU_PANELS=$lp" >> gpurun_out/shard_ab.log
  FEASTLAB_LU_PANELS=$lp timeout 400 python tools/shard_time.py --config 4 --gpus 8 4 2 --steps 2 >> gpurun_out/shard_ab.log 2>&1
done
echo "default" >> gpurun_out/shard_ab.log
timeout 600 python tools/shard_time.py --config 4 --gpus 1 2 4 8 --steps 2 >> gpurun_out/shard_ab.log 2>&1
timeout 400 python tools/shard_time.py --config 4 --gpus 1 2 4 8 --steps 2 --factorization ldlt >> gpurun_out/shard_ab.log 2>&1

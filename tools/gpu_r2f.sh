# r2f: multi-rank bench validation at a non-power-of-two N (padded shards),
# the multi-process tests, and the c5 scaling projection on the final code.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/r2f_multiproc.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_multiproc.log
for cfg in "c2 100000" "c5 4194304"; do
  set -- $cfg
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
     --master-port 29533 bench.py --gpus 2 --exchange host --config $1 --N $2 --steps 5 --warmup 3 \
     --no-per-config --no-cpu-baseline --no-e2e > gpurun_out/r2f_bench2_$1.log 2>&1
  echo "rc=$?" >> gpurun_out/r2f_bench2_$1.log
done
timeout 900 python tools/scaling_projection.py 10 > gpurun_out/r2f_scaling_projection.txt 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "shards or general" > gpurun_out/r2g_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_pytest.log
bash tools/ab_var.sh c5 > gpurun_out/r2g_ab.txt 2>&1
python bench.py --steps 20 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/r2g_bench.log 2>&1

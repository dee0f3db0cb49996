mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "packed or get or host" > gpurun_out/r2h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_pytest.log
python bench.py --steps 20 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/r2h_bench.log 2>&1

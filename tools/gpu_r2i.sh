mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r2i_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_pytest.log
for c in c5 c2 c3; do python tools/level_times.py $c - 10 | grep -E "ms/step|whiten"; done > gpurun_out/r2i_whiten.txt 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench.log 2>&1

# One GPU call: the -m gpu suite (optionally a -k filter), then a short bench.
# Usage: bash tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-chk}
K=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${TAG}_pytest.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
tail -3 gpurun_out/${TAG}_pytest.log

# Round-2 final evidence (r2j, end of the last session): -m gpu suite, full bench line,
# launch list of the bench command, ncu --set full of the c5 factor/backward L0/L1
# launches and the c4 CTA-path factor L0.
set -x
TAG=${1:-r2j}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --quick --no-graph > gpurun_out/${TAG}_ncu_launches.log 2>&1
bash tools/prof_c5.sh 40 2 ${TAG}_c5f 58 2 ${TAG}_c5b
python tools/parity_table.py > gpurun_out/${TAG}_parity.md 2>&1
for c in c5 c2 c3 c1; do python tools/level_times.py $c - 10 | grep -E "ms/step|whiten"; done > gpurun_out/${TAG}_whiten.txt 2>&1
ls -la gpurun_out | tail -30

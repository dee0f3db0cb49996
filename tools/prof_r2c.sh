# Round-2 (session c) evidence on one GPU: the full bench line (per_config),
# the launch list of the bench command, ncu --set full of the c4 CTA-path
# factor L0 (full N) and of its whitening kernel, and the measured parity
# table.  Summaries in base units; no .ncu-rep copied back.
set -x
TAG=${1:-r2c}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --quick --no-graph > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:factor_level -s 15 -c 1 -o gpurun_out/${TAG}_c4f python tools/prof_run.py c4 - 1 > gpurun_out/${TAG}_ncu_c4f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:whiten_evo -s 1 -c 1 -o gpurun_out/${TAG}_c4w python tools/prof_run.py c4 - 1 > gpurun_out/${TAG}_ncu_c4w.log 2>&1
for r in c4f c4w; do
  python tools/ncu_summary.py gpurun_out/${TAG}_$r.ncu-rep > gpurun_out/${TAG}_$r.sum.txt 2>&1
  python tools/ncu_hot.py gpurun_out/${TAG}_$r.ncu-rep 30 0 > gpurun_out/${TAG}_$r.hot0.txt 2>&1
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page raw --csv --print-units base > gpurun_out/${TAG}_$r.raw.csv 2>&1
  rm -f gpurun_out/${TAG}_$r.ncu-rep
done
python tools/parity_table.py > gpurun_out/${TAG}_parity.md 2>&1
du -sh gpurun_out

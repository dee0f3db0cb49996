# Round-2 final evidence (one GPU): the bench line (per_config), the launch
# list of the bench command, ncu --set full of the c5 factor / backward L0 and
# L1 launches, of the c4 factor L0 (full N), and of the large-n path's top
# kernels at n = 500; summaries in base units, raw CSVs, no .ncu-rep (gpurun
# copies back at most 64 MiB).
set -x
TAG=${1:-r2b}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --quick --no-graph > gpurun_out/${TAG}_ncu_launches.log 2>&1
bash tools/prof_c5.sh 40 2 ${TAG}_c5f 58 2 ${TAG}_c5b
ncu --set full --clock-control none --import-source on -k regex:factor_level -s 15 -c 1 -o gpurun_out/${TAG}_c4f python tools/prof_run.py c4 - 1 > gpurun_out/${TAG}_ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"big_qr_panel|big_gemm" -s 400 -c 6 -o gpurun_out/${TAG}_big python tools/big_time.py 64 500 > gpurun_out/${TAG}_ncu_big.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_big_launches.csv python tools/big_time.py 32 500 > gpurun_out/${TAG}_ncu_big_launches.log 2>&1
for r in c4f big; do
  python tools/ncu_summary.py gpurun_out/${TAG}_$r.ncu-rep > gpurun_out/${TAG}_$r.sum.txt 2>&1
  python tools/ncu_hot.py gpurun_out/${TAG}_$r.ncu-rep 30 0 > gpurun_out/${TAG}_$r.hot0.txt 2>&1
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page raw --csv --print-units base > gpurun_out/${TAG}_$r.raw.csv 2>&1
  rm -f gpurun_out/${TAG}_$r.ncu-rep
done
du -sh gpurun_out

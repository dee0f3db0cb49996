# Session-c profile capture (one GPU): bench line, launch list, ncu --set full of
# the c5 factor L0/L1 launches and the c4 CTA-path factor, all configs.
set -x
python bench.py > gpurun_out/bench_c.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c.csv \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_launches.log 2>&1
bash tools/prof_c5.sh 40 2 rc_factor
python tools/prof_run.py c4 2000 > gpurun_out/plain_c4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:factor_level -s 0 -c 1 -o gpurun_out/rc_c4factor python tools/prof_run.py c4 2000 > gpurun_out/ncu_c4.log 2>&1
python tools/all_configs.py > gpurun_out/all_c.txt 2>&1
du -sh gpurun_out

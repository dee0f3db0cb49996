# Round profile capture (one GPU): launch list of a bench step + ncu --set full
# of the c5 dominant launches and the c4 CTA-path factor.  Output: gpurun_out/
set -x
python bench.py --steps 2 --warmup 3 --quick > gpurun_out/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_launches.log 2>&1
python tools/prof_run.py c5 > gpurun_out/plain_c5.log 2>&1 || exit 1
K='regex:small_factor|small_backward'
ncu --set full --clock-control none --import-source on -k $K -s 40 -c 2 -o gpurun_out/rb_factor python tools/prof_run.py c5 > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k $K -s 58 -c 2 -o gpurun_out/rb_backward python tools/prof_run.py c5 > gpurun_out/ncu_b.log 2>&1
python tools/prof_run.py c4 2000 > gpurun_out/plain_c4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:factor_level -s 0 -c 1 -o gpurun_out/rb_c4factor python tools/prof_run.py c4 2000 > gpurun_out/ncu_c4.log 2>&1
du -sh gpurun_out

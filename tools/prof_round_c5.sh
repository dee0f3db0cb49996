# ncu --set full of the c5 dominant launches (indices: see tools/prof_c5.sh)
set -x
python tools/prof_run.py c5 > gpurun_out/plain_c5.log 2>&1 || exit 1
K='regex:small_factor|small_backward'
ncu --set full --clock-control none --import-source on -k $K -s 40 -c 2 -o gpurun_out/rb_factor python tools/prof_run.py c5 > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k $K -s 58 -c 2 -o gpurun_out/rb_backward python tools/prof_run.py c5 > gpurun_out/ncu_b.log 2>&1

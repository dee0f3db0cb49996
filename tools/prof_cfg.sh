# ncu --set full of selected kernel launches of one config (tools/prof_run.py):
#   prof_cfg.sh CONFIG N KERNEL_REGEX SKIP COUNT NAME
set -x
python tools/prof_run.py $1 $2 > gpurun_out/plain_$6.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c $5 -o gpurun_out/$6 python tools/prof_run.py $1 $2 > gpurun_out/ncu_$6.log 2>&1
python tools/ncu_summary.py gpurun_out/$6.ncu-rep > gpurun_out/$6.sum.txt 2>&1
python tools/ncu_hot.py gpurun_out/$6.ncu-rep 40 0 > gpurun_out/$6.hot0.txt 2>&1

# ncu --set full of selected launches of a c5 run (see tools/prof_run.py):
#   prof_c5.sh SKIP COUNT NAME  (launch indices among small_factor|small_backward kernels;
#   after 2 warm-up runs of c5 (20 matching launches per run: factor L0..L7, subtree pass,
#   tail; backward tail, subtree pass, L7..L0): factor L0 = 40, L1 = 41, backward L1 = 58, L0 = 59)
set -x
python tools/prof_run.py c5 > gpurun_out/plain.log 2>&1 || exit 1
K='regex:small_factor|small_backward'
while [ $# -ge 3 ]; do
  ncu --set full --clock-control none --import-source on -k $K -s $1 -c $2 -o gpurun_out/$3 python tools/prof_run.py c5 > gpurun_out/ncu_$3.log 2>&1
  python tools/ncu_summary.py gpurun_out/$3.ncu-rep > gpurun_out/$3.sum.txt 2>&1
  python tools/ncu_hot.py gpurun_out/$3.ncu-rep 30 0 > gpurun_out/$3.hot0.txt 2>&1
  python tools/ncu_hot.py gpurun_out/$3.ncu-rep 30 1 > gpurun_out/$3.hot1.txt 2>&1
  ncu -i gpurun_out/$3.ncu-rep --page raw --csv --print-units base > gpurun_out/$3.raw.csv 2>&1
  rm -f gpurun_out/$3.ncu-rep   # (gpurun copies back at most 64 MiB)
  shift 3
done
du -sh gpurun_out

# A/B: c5 per-level times + backward L0 DRAM bytes for every variant
for v in paper_2502_11686_b200/variants/libks_*.so; do
  echo "=== $v"
  KS_LIB=$PWD/$v python tools/level_times.py c5 - 10 | grep -E "ms/step|backward L= [0-3] "
  KS_LIB=$PWD/$v ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --print-units base --csv -k regex:small_backward_tma -s 16 -c 2 python tools/prof_run.py c5 - 1 2>/dev/null | grep -E "dram|duration" | cut -d, -f12- | head -6
done

# A/B: sum-of-launches step time of configs for the default build and every variant
mkdir -p gpurun_out
for i in 1 2; do
  for c in "$@"; do
    echo "=== default $c"; python tools/level_times.py $c - 10 | grep -E "ms/step|factor   L= [0-3] |backward L= [0-1] "
    for v in paper_2502_11686_b200/variants/libks_*.so; do
      echo "=== $v $c"; KS_LIB=$PWD/$v python tools/level_times.py $c - 10 | grep -E "ms/step|factor   L= [0-3] |backward L= [0-1] "
    done
  done
done

# A/B over several configs: per-level times of every built variant (tools/level_times.py)
for v in paper_2502_11686_b200/variants/libks_*.so; do
  for c in "$@"; do
    echo "=== $v $c"; KS_LIB=$PWD/$v python tools/level_times.py $c - 10 | grep -E "ms/step|L= [0-3] |L=1[0-2]"
  done
done

# A/B: per-level times of one config for every built variant (tools/level_times.py)
for v in paper_2502_11686_b200/variants/libks_*.so; do
  echo "=== $v"; KS_LIB=$PWD/$v python tools/level_times.py ${1:-c5} ${2:--} 5 | grep -E "ms/step|L= [0-3] |L=1[0-2]"
done

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for K in 64 32 16 8 4 2; do
  echo "=== K=$K"
  PPRG_COLUMNS=$K timeout 300 python tools/profile_one.py --queries 64 --reps 2
done

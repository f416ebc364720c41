#!/bin/bash
# A/B of library variants on one-source (K=1) PowerPush: scale 22 (configs[2] graph),
# scale 25 (configs[4] graph), scale 17 (configs[0]). usage: bash tools/k1ab.sh ARM...
for v in "$@"; do
  if [ $v = main ]; then lib=""; else lib=libv_$v/libpprg.so; fi
  echo "== $v"; PPRG_LIB=$lib python tools/profile_one.py --queries 1 --reps 2 | tail -1 | cut -c1-110
  PPRG_LIB=$lib python tools/profile_one.py --queries 1 --reps 1 --scale 25 --ef 32 --seed 5 | tail -1 | cut -c1-110
  PPRG_LIB=$lib python tools/profile_one.py --queries 1 --reps 3 --scale 17 --ef 8 --seed 1 | tail -1 | cut -c1-110
done

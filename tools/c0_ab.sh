#!/bin/bash
# configs[0] (one source, R-MAT 17/8) under narrow-path grid / tile shapes
for lib in "" libv_u4/libpprg.so; do
  for tpb in 1 2 4 8; do
    echo "== lib=${lib:-main} TILES_PER_BLOCK=$tpb"
    PPRG_LIB=$lib PPRG_TILES_PER_BLOCK=$tpb python tools/profile_one.py --queries 1 --reps 3 --scale 17 --ef 8 --seed 1 | tail -1 | cut -c1-130
  done
done

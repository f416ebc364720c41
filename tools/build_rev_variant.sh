#!/bin/bash
# Build libv_<name>/libpprg.so from the engine sources of git revision <rev>
# (A/B baselines on the GPU box: PPRG_LIB=libv_<name>/libpprg.so).
# usage: tools/build_rev_variant.sh <name> <rev> ["<extra nvcc flags>"]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$2" paper_2101_03652_b200/csrc include | tar -x -C "$TMP"
OUT=$ROOT/libv_$1; mkdir -p "$OUT/obj"
for f in "$TMP"/paper_2101_03652_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $3 -c "$f" -o "$OUT/obj/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libpprg.so" "$OUT"/obj/*.o
rm -rf "$OUT/obj" "$TMP"

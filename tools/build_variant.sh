#!/bin/bash
# Build a variant of libpprg.so with extra nvcc flags into libv_<name>/ (for A/B
# timing on the GPU box; select it with PPRG_LIB=libv_<name>/libpprg.so).
# usage: tools/build_variant.sh <name> "<extra flags>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/libv_$1; mkdir -p "$OUT/obj"
for f in "$ROOT"/paper_2101_03652_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr $2 -c "$f" -o "$OUT/obj/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libpprg.so" "$OUT"/obj/*.o
rm -rf "$OUT/obj"

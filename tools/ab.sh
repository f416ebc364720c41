#!/bin/bash
# A/B timing on configs[2] (64 columns), two rounds: bash tools/ab.sh ARM...
# ARM = main (lib/libpprg.so) | <name> (libv_<name>/libpprg.so) | VAR=value[,VAR=value] (env, main lib)
for round in 1 2; do
  for v in "$@"; do
    lib=""; envs=""
    if [[ "$v" == *=* ]]; then envs=${v//,/ }; elif [ "$v" != main ]; then lib=libv_$v/libpprg.so; fi
    echo "=== $v"
    env PPRG_LIB=$lib $envs timeout 300 python tools/profile_one.py --queries 64 --reps 2 2>&1 | grep wall | tail -1
  done
done

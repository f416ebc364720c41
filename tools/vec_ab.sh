for K in 64 32 16 8 4; do for v in novec main; do
  if [ $v = main ]; then lib=""; else lib=libv_$v/libpprg.so; fi
  echo "== K=$K $v"; PPRG_COLUMNS=$K PPRG_LIB=$lib timeout 300 python tools/profile_one.py --queries 64 --reps 2 | tail -1 | cut -c1-75
done; done

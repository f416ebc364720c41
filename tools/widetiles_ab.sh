for v in "PPRG_WIDE_TILES=0" "PPRG_WIDE_TILES=2" "PPRG_WIDE_TILES=1" "PPRG_WIDE_TILES=4"; do
  echo "== $v"
  env $v python tools/profile_one.py --queries 64 --reps 2 --scale 17 --ef 8 --seed 1 | tail -1 | cut -c1-150
  env $v python tools/profile_one.py --queries 64 --reps 1 | tail -1 | cut -c1-100
done

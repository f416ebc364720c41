for f in 1 0.5 0.25 0.125; do
PPRG_GRID_FRAC=$f timeout 300 python tools/ab_quick.py 0,1 > gpurun_out/c18_frac$f.json 2>&1
done
for f in gpurun_out/c18_*.json; do echo $f; tail -1 $f; done

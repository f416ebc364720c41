for h in 0.03125 0.015625 0.0078125 0.00390625; do
PPRG_REFINE_HANDOFF=$h timeout 300 python tools/ab_quick.py 3 > gpurun_out/c21_h$h.json 2>&1
done
for d in 8 32; do
PPRG_SPP_SCAN_DIV=$d timeout 300 python tools/ab_quick.py 3 > gpurun_out/c21_d$d.json 2>&1
done
for f in gpurun_out/c21_*.json; do echo $f; tail -1 $f; done

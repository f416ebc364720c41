python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/c22_smoke.log 2>&1; tail -2 gpurun_out/c22_smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/c22_ref.json 2> gpurun_out/c22_ref.err; tail -c 500 gpurun_out/c22_ref.json
for c in 64 32; do
for d in 16 32; do
PPRG_SPP_COLUMNS=$c PPRG_SPP_SCAN_DIV=$d timeout 300 python tools/ab_quick.py 3 > gpurun_out/c22_spp_c${c}_d$d.json 2>&1
PPRG_SPP_COLUMNS=$c PPRG_SPP_SCAN_DIV=$d timeout 300 python tools/ab_quick.py 3 > gpurun_out/c22_spp_c${c}_d${d}_b.json 2>&1
done
done
for f in gpurun_out/c22_spp*.json; do echo $f; tail -1 $f | cut -c1-250; done

export PPRG_DELTA=1
timeout 300 python tools/ab_quick.py 2 > gpurun_out/c29_base.json 2>&1; tail -1 gpurun_out/c29_base.json | cut -c1-330
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsweeps -c 1 \
  -o gpurun_out/c29_dsweep python tools/profile_one.py --queries 64 > gpurun_out/c29_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/c29_ncu.log

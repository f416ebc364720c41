timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dsweeps -c 1 \
  -o gpurun_out/c52_dsweep python tools/profile_one.py --queries 64 > gpurun_out/c52_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/c52_ncu.log

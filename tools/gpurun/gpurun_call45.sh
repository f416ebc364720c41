timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_delta.py -x -q -k "speedppr or config3 or delta" > gpurun_out/c45_spp.log 2>&1
echo "spp rc=$?"; tail -4 gpurun_out/c45_spp.log
PPRG_DELTA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "speedppr or refine or mc" > gpurun_out/c45_spp1.log 2>&1
echo "spp forced rc=$?"; tail -4 gpurun_out/c45_spp1.log
for i in 1 2; do
PPRG_DELTA_REFINE=0 timeout 300 python tools/ab_quick.py 3 2>&1 | tail -1 | cut -c1-400
timeout 300 python tools/ab_quick.py 3 2>&1 | tail -1 | cut -c1-400
done
PPRG_DELTA=1 timeout 300 python tools/ab_quick.py 1 2>&1 | tail -1 | cut -c1-400
PPRG_DELTA=0 timeout 300 python tools/ab_quick.py 1 2>&1 | tail -1 | cut -c1-400

timeout 900 python -m pytest tests/test_gpu_delta.py tests/test_gpu_fuzz.py -x -q > gpurun_out/c50_delta.log 2>&1
echo "delta rc=$?"; tail -4 gpurun_out/c50_delta.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config2" > gpurun_out/c50_cfg.log 2>&1
echo "cfg rc=$?"; tail -3 gpurun_out/c50_cfg.log
for i in 1 2; do timeout 300 python tools/ab_quick.py 2 2>&1 | tail -1 | cut -c1-330; done
python tools/k32_probe.py | tail -1

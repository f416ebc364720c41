# delta sweeps: first correctness + timing
export PPRG_DELTA=1
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c25_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -15 gpurun_out/c25_fuzz.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config1_power_push or config2" > gpurun_out/c25_cfg.log 2>&1
echo "cfg rc=$?"; tail -15 gpurun_out/c25_cfg.log
timeout 300 python tools/ab_quick.py 2 > gpurun_out/c25_delta.json 2> gpurun_out/c25_delta.err; tail -1 gpurun_out/c25_delta.json | cut -c1-400; tail -3 gpurun_out/c25_delta.err
PPRG_DELTA=0 timeout 300 python tools/ab_quick.py 2 > gpurun_out/c25_old.json 2>&1; tail -1 gpurun_out/c25_old.json | cut -c1-400

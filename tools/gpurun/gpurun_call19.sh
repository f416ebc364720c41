timeout 900 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_determinism.py -x -q > gpurun_out/c19_pytest.log 2>&1
tail -3 gpurun_out/c19_pytest.log
for l in 1 2 4; do PPRG_LANES=$l timeout 300 python tools/concurrency_probe.py > gpurun_out/c19_conc_lanes$l.json 2>&1; tail -1 gpurun_out/c19_conc_lanes$l.json; done
timeout 300 python tools/ab_quick.py 0,1,2 > gpurun_out/c19_ab.json 2>&1; tail -1 gpurun_out/c19_ab.json

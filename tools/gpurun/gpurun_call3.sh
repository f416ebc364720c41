timeout 300 python tools/ab_quick.py > gpurun_out/c3_ab_dev.json 2> gpurun_out/c3_ab_dev.err
PPRG_HOST_LEVELS=1 timeout 300 python tools/ab_quick.py > gpurun_out/c3_ab_host.json 2> gpurun_out/c3_ab_host.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/c3_pytest.log 2>&1
tail -3 gpurun_out/c3_pytest.log

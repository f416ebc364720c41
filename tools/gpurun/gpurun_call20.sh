timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c20_pytest.log 2>&1
tail -3 gpurun_out/c20_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/c20_bench.json 2> gpurun_out/c20_bench.err
tail -c 400 gpurun_out/c20_bench.json

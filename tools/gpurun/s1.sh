python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/s1_smoke.log 2>&1; tail -n 2 gpurun_out/s1_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.log 2>&1; tail -n 3 gpurun_out/s1_pytest.log
timeout 600 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err; tail -c 600 gpurun_out/s1_bench.json

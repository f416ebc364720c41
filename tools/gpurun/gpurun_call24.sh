# re-entry baseline: whole GPU suite + bench line
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c24_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/c24_pytest.log
timeout 900 python bench.py > gpurun_out/c24_bench.json 2> gpurun_out/c24_bench.err
echo "bench rc=$?"; cut -c1-1500 gpurun_out/c24_bench.json

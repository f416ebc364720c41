set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/microbench/dump_transpose.py /tmp/transpose.bin > gpurun_out/c1_dump.log 2>&1
timeout 600 tools/microbench/nk /tmp/transpose.bin > gpurun_out/c1_nk.log 2>&1
timeout 300 tools/microbench/ge /tmp/transpose.bin > gpurun_out/c1_ge.log 2>&1
timeout 600 python bench.py > gpurun_out/c1_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c1_pytest.log 2>&1
echo done

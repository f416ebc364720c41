timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c8_pytest.log 2>&1
tail -3 gpurun_out/c8_pytest.log
bash tools/round_profile.sh r02a > gpurun_out/c8_round.log 2>&1
tail -5 gpurun_out/c8_round.log
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-secondary > gpurun_out/c8_bench_g2.json 2> gpurun_out/c8_bench_g2.err
tail -c 600 gpurun_out/c8_bench_g2.json

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c16_pytest.log 2>&1
tail -3 gpurun_out/c16_pytest.log
bash tools/round_profile.sh r02b > gpurun_out/c16_round.log 2>&1
tail -3 gpurun_out/c16_round.log

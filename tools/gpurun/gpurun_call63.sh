# full GPU suite with the delta sweeps as the configs[2] default, then the round profile
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c63_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/c63_pytest.log
bash tools/round_profile.sh r02f

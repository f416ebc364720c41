export PPRG_DELTA=1
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_delta.py -x -q -k "dead_end or (vs_oracle and 3000-4-700-5-64) or (vs_oracle and 300-1-3000-2-32)" > gpurun_out/c56_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -6 gpurun_out/c56_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_delta.py -x -q -k "dead_end or (vs_oracle and 300-1-3000-2-32)" > gpurun_out/c56_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -6 gpurun_out/c56_racecheck.log

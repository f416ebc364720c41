#!/bin/bash
# GPU iteration helper: parity suite, then the configs[2] 64-column timing.
# usage (under gpurun): bash tools/perf_check.sh TAG [pytest-args...]
tag=${1:-run}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
timeout 300 python tools/profile_one.py --queries 64 --reps 3 > gpurun_out/${tag}_perf.log 2>&1
cat gpurun_out/${tag}_perf.log

#!/bin/bash
# Bench line + ncu launch list + one --set full capture of the sweep kernel.
# usage (under gpurun): bash tools/round_profile.sh TAG
tag=${1:-v}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
echo "bench rc=$?"; cat gpurun_out/bench_${tag}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  --e2e-steps 1 > gpurun_out/launches_${tag}.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_dsweeps|k_sweeps" -c 1 \
  -o gpurun_out/sweep_${tag} python tools/profile_one.py --queries 64 > gpurun_out/sweep_${tag}.log 2>&1
echo "ncu rc=$?"

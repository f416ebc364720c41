timeout 900 python -m pytest tests/test_gpu_delta.py -x -q > gpurun_out/c42_delta.log 2>&1
echo "delta rc=$?"; tail -12 gpurun_out/c42_delta.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c42_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c42_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3), d)")"; }
run auto
timeout 900 python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c42_bench.json 2> gpurun_out/c42_bench.err; cut -c1-1800 gpurun_out/c42_bench.json; tail -3 gpurun_out/c42_bench.err

run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c59_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c59_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
for r in 1 2; do
run base_$r
for v in s96 s128 s40; do run ${v}_$r PPRG_LIB=$PWD/libv_$v/libpprg.so; done
done
run t256 PPRG_DS_TASK=256
run t160 PPRG_DS_TASK=160
run p384 PPRG_DS_PIECE=384
python tools/k32_probe.py | tail -1
timeout 600 python -m pytest tests/test_gpu_delta.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2

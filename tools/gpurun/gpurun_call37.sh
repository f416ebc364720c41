export PPRG_DELTA=1
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c37_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c37_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'])")"; }
for v in g8b4 g6b4 g6b5 g8b3; do run $v PPRG_LIB=$PWD/libv_$v/libpprg.so; done
run g6b5_fuzz PPRG_LIB=$PWD/libv_g6b5/libpprg.so
PPRG_LIB=$PWD/libv_g6b5/libpprg.so timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" 2>&1 | tail -2
PPRG_LIB=$PWD/libv_g8b4/libpprg.so timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" 2>&1 | tail -2

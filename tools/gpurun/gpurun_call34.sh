export PPRG_DELTA=1
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c34_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c34_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'])")"; }
for v in h0p1 h1p0 h0p0 h0p0l0; do run $v PPRG_LIB=$PWD/libv_$v/libpprg.so; done
run h0p0_again PPRG_LIB=$PWD/libv_h0p0/libpprg.so

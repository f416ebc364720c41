run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c66_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c66_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
run base
for v in b6g6l0 b6g8l0 b5l0; do run ${v} PPRG_LIB=$PWD/libv_$v/libpprg.so; done

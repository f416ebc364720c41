export PPRG_DELTA=1
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c40_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c40_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
run w1 PPRG_DS_WAVES=1
run w32l32 PPRG_DS_WAVES=32 PPRG_DS_LAG=32
run w32l8 PPRG_DS_WAVES=32 PPRG_DS_LAG=8
run w32l4 PPRG_DS_WAVES=32 PPRG_DS_LAG=4
run w64l4 PPRG_DS_WAVES=64 PPRG_DS_LAG=4
run w64l6 PPRG_DS_WAVES=64 PPRG_DS_LAG=6
run w16l1 PPRG_DS_WAVES=16 PPRG_DS_LAG=1
run w8l1 PPRG_DS_WAVES=8 PPRG_DS_LAG=1

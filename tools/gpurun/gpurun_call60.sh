run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c60_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c60_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
run l5 PPRG_DS_LAG=5
run l7 PPRG_DS_LAG=7
run w48l5 PPRG_DS_WAVES=48 PPRG_DS_LAG=5
run w56l5 PPRG_DS_WAVES=56 PPRG_DS_LAG=5
run w64l6 
run w40l4 PPRG_DS_WAVES=40 PPRG_DS_LAG=4
run scan64 PPRG_DS_SCAN_DIV=64
run scan512 PPRG_DS_SCAN_DIV=512

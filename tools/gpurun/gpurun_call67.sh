run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c67_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c67_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
run l4 PPRG_DS_LAG=4
run l4p256 PPRG_DS_LAG=4 PPRG_DS_PIECE=256
run l4p128 PPRG_DS_LAG=4 PPRG_DS_PIECE=128
run l4t96 PPRG_DS_LAG=4 PPRG_DS_TASK=96
run l4t96p128 PPRG_DS_LAG=4 PPRG_DS_TASK=96 PPRG_DS_PIECE=128
run l3t96p128 PPRG_DS_LAG=3 PPRG_DS_TASK=96 PPRG_DS_PIECE=128
run l6t96p128 PPRG_DS_TASK=96 PPRG_DS_PIECE=128

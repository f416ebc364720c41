run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c53_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c53_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
run base
run l5 PPRG_DS_LAG=5
run l4 PPRG_DS_LAG=4
run l8 PPRG_DS_LAG=8
run w48l4 PPRG_DS_WAVES=48 PPRG_DS_LAG=4
run w32l3 PPRG_DS_WAVES=32 PPRG_DS_LAG=3
run p256 PPRG_DS_PIECE=256
run p384 PPRG_DS_PIECE=384
run t384 PPRG_DS_TASK=384
run t192 PPRG_DS_TASK=192
run base2

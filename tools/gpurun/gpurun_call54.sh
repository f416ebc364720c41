run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c54_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c54_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
for r in 1 2; do
run t128_$r PPRG_DS_TASK=128
run t160_$r PPRG_DS_TASK=160
run t192_$r PPRG_DS_TASK=192
run t256_$r PPRG_DS_TASK=256
run t192p384_$r PPRG_DS_TASK=192 PPRG_DS_PIECE=384
done

export PPRG_DELTA=1 PPRG_DS_WAVES=64 PPRG_DS_LAG=6
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c41_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -2 gpurun_out/c41_fuzz.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config1_power_push or config2" > gpurun_out/c41_cfg.log 2>&1
echo "cfg rc=$?"; tail -2 gpurun_out/c41_cfg.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c41_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c41_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'], round(d['sweep_ms']/d['max_sweeps'],3))")"; }
run base
for v in s64 s16 s64g4; do run $v PPRG_LIB=$PWD/libv_$v/libpprg.so; done
run w64l5 PPRG_DS_LAG=5
run w48l4 PPRG_DS_WAVES=48 PPRG_DS_LAG=4
run w64l8 PPRG_DS_LAG=8

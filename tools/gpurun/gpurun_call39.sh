export PPRG_DELTA=1
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c39_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -2 gpurun_out/c39_fuzz.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config1_power_push or config2" > gpurun_out/c39_cfg.log 2>&1
echo "cfg rc=$?"; tail -2 gpurun_out/c39_cfg.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c39_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c39_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'])")"; }
run base
run w24 PPRG_DS_WAVES=24
run w32 PPRG_DS_WAVES=32
run w32l3 PPRG_DS_WAVES=32 PPRG_DS_LAG=3
run w48l3 PPRG_DS_WAVES=48 PPRG_DS_LAG=3
run w12 PPRG_DS_WAVES=12
run p256 PPRG_DS_PIECE=256
run t128 PPRG_DS_TASK=128

export PPRG_DELTA=1
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c35_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -3 gpurun_out/c35_fuzz.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config1_power_push or config2" > gpurun_out/c35_cfg.log 2>&1
echo "cfg rc=$?"; tail -3 gpurun_out/c35_cfg.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c35_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c35_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'])")"; }
run base
run pfrows PPRG_LIB=$PWD/libv_pfrows/libpprg.so
run minb6 PPRG_LIB=$PWD/libv_minb6/libpprg.so
run p256 PPRG_DS_PIECE=256
run t512 PPRG_DS_TASK=512
run w24 PPRG_DS_WAVES=24
run pfrows_w24 PPRG_DS_WAVES=24 PPRG_LIB=$PWD/libv_pfrows/libpprg.so

export PPRG_DELTA=1
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c27_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -3 gpurun_out/c27_fuzz.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config1_power_push or config2" > gpurun_out/c27_cfg.log 2>&1
echo "cfg rc=$?"; tail -3 gpurun_out/c27_cfg.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c27_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c27_$tag.json | cut -c1-330)"; }
run base
run w16 PPRG_DS_WAVES=16
run w64 PPRG_DS_WAVES=64
run l3 PPRG_DS_LAG=3
run w64l3 PPRG_DS_WAVES=64 PPRG_DS_LAG=3
run t1k PPRG_DS_TILE=1024
run t4k PPRG_DS_TILE=4096

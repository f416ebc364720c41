export PPRG_DELTA=1
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c30_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -3 gpurun_out/c30_fuzz.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config1_power_push or config2" > gpurun_out/c30_cfg.log 2>&1
echo "cfg rc=$?"; tail -3 gpurun_out/c30_cfg.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c30_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c30_$tag.json | cut -c1-330)"; }
run base
run t128 PPRG_DS_TASK=128
run t512 PPRG_DS_TASK=512
run p512 PPRG_DS_PIECE=512
run p2k PPRG_DS_PIECE=2048
run w16 PPRG_DS_WAVES=16
run w64 PPRG_DS_WAVES=64

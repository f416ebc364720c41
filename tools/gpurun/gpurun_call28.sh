export PPRG_DELTA=1
timeout 600 python -m pytest tests/test_gpu_fuzz.py -x -q -k "power_push_fuzz" > gpurun_out/c28_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -3 gpurun_out/c28_fuzz.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c28_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c28_$tag.json | cut -c1-330)"; }
run base
run minb3 PPRG_LIB=$PWD/libv_minb3/libpprg.so
run minb5 PPRG_LIB=$PWD/libv_minb5/libpprg.so
run w16 PPRG_DS_WAVES=16
run w24 PPRG_DS_WAVES=24

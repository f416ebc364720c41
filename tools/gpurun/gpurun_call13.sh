timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fuzz.py tests/test_gpu_determinism.py -x -q > gpurun_out/c13_pytest.log 2>&1
tail -3 gpurun_out/c13_pytest.log
for i in 1 2; do
PPRG_LIB=$PWD/libv_vec2/libpprg.so timeout 300 python tools/ab_quick.py 2,3 > gpurun_out/c13_ab_vec2_$i.json 2>&1
timeout 300 python tools/ab_quick.py 2,3 > gpurun_out/c13_ab_vec4_$i.json 2>&1
PPRG_COLUMNS=32 timeout 300 python tools/ab_quick.py 2 > gpurun_out/c13_ab_vec4_k32_$i.json 2>&1
PPRG_COLUMNS=32 PPRG_LIB=$PWD/libv_vec2/libpprg.so timeout 300 python tools/ab_quick.py 2 > gpurun_out/c13_ab_vec2_k32_$i.json 2>&1
done
for f in gpurun_out/c13_ab*.json; do echo $f; tail -1 $f; done

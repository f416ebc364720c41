timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -x -q -k "speedppr or mc or monte or determin or walk" > gpurun_out/c23_pytest.log 2>&1
tail -3 gpurun_out/c23_pytest.log
for i in 1 2; do
PPRG_LIB=$PWD/libv_prev/libpprg.so timeout 300 python tools/ab_quick.py 3 > gpurun_out/c23_prev$i.json 2>&1
timeout 300 python tools/ab_quick.py 3 > gpurun_out/c23_new$i.json 2>&1
done
for f in gpurun_out/c23_*.json; do echo $f; tail -1 $f | cut -c1-300; done

timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_reference_acceptance.py -x -q > gpurun_out/c7_det.log 2>&1
tail -5 gpurun_out/c7_det.log
for i in 1 2; do
PPRG_LIB=$PWD/paper_2101_03652_b200/libv_head/libpprg.so timeout 300 python tools/ab_quick.py 0,2,3 > gpurun_out/c7_ab_head$i.json 2>&1
for gl in 32 8 4; do
PPRG_DRAIN_GL=$gl timeout 300 python tools/ab_quick.py 0,2,3 > gpurun_out/c7_ab_gl${gl}_$i.json 2>&1
done
done
AB_DET=1 timeout 600 python tools/ab_quick.py > gpurun_out/c7_ab_det.json 2> gpurun_out/c7_ab_det.err
for f in gpurun_out/c7_ab_*.json; do echo $f; cat $f; done

timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_reference_acceptance.py -x -q > gpurun_out/c5_det.log 2>&1
tail -5 gpurun_out/c5_det.log
timeout 300 python tools/ab_quick.py > gpurun_out/c5_ab_fast.json 2> gpurun_out/c5_ab_fast.err
AB_DET=1 timeout 600 python tools/ab_quick.py > gpurun_out/c5_ab_det.json 2> gpurun_out/c5_ab_det.err
cat gpurun_out/c5_ab_fast.json gpurun_out/c5_ab_det.json

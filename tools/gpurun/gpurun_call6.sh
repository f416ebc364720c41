timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_reference_acceptance.py -x -q > gpurun_out/c6_det.log 2>&1
tail -5 gpurun_out/c6_det.log
for i in 1 2; do
PPRG_LIB=$PWD/paper_2101_03652_b200/libv_head/libpprg.so timeout 300 python tools/ab_quick.py 0,2 > gpurun_out/c6_ab_head$i.json 2>&1
timeout 300 python tools/ab_quick.py 0,2 > gpurun_out/c6_ab_new$i.json 2>&1
done
AB_DET=1 timeout 600 python tools/ab_quick.py > gpurun_out/c6_ab_det.json 2> gpurun_out/c6_ab_det.err
cat gpurun_out/c6_ab_*.json
timeout 600 tools/microbench/ge /tmp/transpose.bin > gpurun_out/c6_ge.log 2>&1 || (python tools/microbench/dump_transpose.py /tmp/transpose.bin > /dev/null 2>&1; timeout 600 tools/microbench/ge /tmp/transpose.bin > gpurun_out/c6_ge.log 2>&1)

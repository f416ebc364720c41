for i in 1 2; do
PPRG_LIB=$PWD/paper_2101_03652_b200/libv_head/libpprg.so timeout 300 python tools/ab_quick.py > gpurun_out/c12_ab_head$i.json 2>&1
timeout 300 python tools/ab_quick.py > gpurun_out/c12_ab_new$i.json 2>&1
done
for wv in 4 8 16; do
AB_DET=1 PPRG_DET_WAVES=$wv timeout 600 python tools/ab_quick.py 0,2 > gpurun_out/c12_ab_det_w$wv.json 2>&1
done
python tools/microbench/dump_transpose.py /tmp/transpose.bin > /dev/null 2>&1
timeout 600 tools/microbench/nk /tmp/transpose.bin > gpurun_out/c12_nk.log 2>&1
for f in gpurun_out/c12_ab*.json; do echo $f; tail -1 $f; done
head -12 gpurun_out/c12_nk.log

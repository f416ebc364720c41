timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c11_pytest.log 2>&1
tail -3 gpurun_out/c11_pytest.log
for i in 1 2; do
PPRG_LIB=$PWD/paper_2101_03652_b200/libv_head/libpprg.so timeout 300 python tools/ab_quick.py > gpurun_out/c11_ab_head$i.json 2>&1
timeout 300 python tools/ab_quick.py > gpurun_out/c11_ab_new$i.json 2>&1
done
AB_DET=1 timeout 600 python tools/ab_quick.py > gpurun_out/c11_ab_det.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c11_launches.csv python tools/ab_quick.py 2 > /dev/null 2>&1
for f in gpurun_out/c11_ab*.json; do echo $f; tail -1 $f; done

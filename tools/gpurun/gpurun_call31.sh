export PPRG_DELTA=1
run() { tag=$1; shift; env "$@" timeout 300 python tools/ab_quick.py 2 > gpurun_out/c31_$tag.json 2>&1; echo "$tag $(tail -1 gpurun_out/c31_$tag.json | python -c "
import sys,json
d=json.loads(sys.stdin.read())['configs[2] 64-block']; print(round(d['sweep_ms'],1), d['max_sweeps'])")"; }
run p512w16 PPRG_DS_PIECE=512 PPRG_DS_WAVES=16
run p256w16 PPRG_DS_PIECE=256 PPRG_DS_WAVES=16
run p256w32 PPRG_DS_PIECE=256 PPRG_DS_WAVES=32
run p256w24 PPRG_DS_PIECE=256 PPRG_DS_WAVES=24
run p256w32l3 PPRG_DS_PIECE=256 PPRG_DS_WAVES=32 PPRG_DS_LAG=3
run p256w48l3 PPRG_DS_PIECE=256 PPRG_DS_WAVES=48 PPRG_DS_LAG=3
run p256w8 PPRG_DS_PIECE=256 PPRG_DS_WAVES=8
run p256w16_minb6 PPRG_DS_PIECE=256 PPRG_DS_WAVES=16 PPRG_LIB=$PWD/libv_minb6/libpprg.so
run p256w16_minb8 PPRG_DS_PIECE=256 PPRG_DS_WAVES=16 PPRG_LIB=$PWD/libv_minb8/libpprg.so
run p256w16_pipe4 PPRG_DS_PIECE=256 PPRG_DS_WAVES=16 PPRG_LIB=$PWD/libv_pipe4/libpprg.so
run p512w16_pipe4 PPRG_DS_PIECE=512 PPRG_DS_WAVES=16 PPRG_LIB=$PWD/libv_pipe4/libpprg.so
run p256w16t512 PPRG_DS_PIECE=512 PPRG_DS_WAVES=16 PPRG_DS_TASK=512

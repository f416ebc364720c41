PPRG_DEBUG_LOCAL=1 timeout 300 python tools/profile_speedppr.py > gpurun_out/c4_spp_levels.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c4_spp_launches.csv python tools/profile_speedppr.py > gpurun_out/c4_spp_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_drain|k_mc_entries|k_mc_big|k_index" -c 8 \
  -o gpurun_out/c4_spp_full python tools/profile_speedppr.py > gpurun_out/c4_spp_full.log 2>&1
echo done

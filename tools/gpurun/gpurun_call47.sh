timeout 900 python bench.py > gpurun_out/c47_bench.json 2> gpurun_out/c47_bench.err
echo "bench rc=$?"; cut -c1-600 gpurun_out/c47_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/c47_ref.json 2> gpurun_out/c47_ref.err
echo "ref rc=$?"; cut -c1-600 gpurun_out/c47_ref.json
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/c47_g2.json 2> gpurun_out/c47_g2.err
echo "g2 rc=$?"; cut -c1-600 gpurun_out/c47_g2.json; tail -2 gpurun_out/c47_g2.err

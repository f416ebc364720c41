for h in 0.0078125 0.004 0.002 0.001 0.0005 0.0001; do
echo "handoff $h"; PPRG_REFINE_HANDOFF=$h timeout 300 python tools/ab_quick.py 3 2>&1 | tail -1 | cut -c40-400
done

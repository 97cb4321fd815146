# A/B: warp-per-candidate vs thread-per-candidate simulate kernel (dev tool)
for rep in 1 2; do
for t in 0 1; do echo "== HESP_SIM_THREAD=$t"; HESP_SIM_THREAD=$t python scripts/probe_throughput.py C2 100000 2>&1 | tail -1 | sed "s/statuses.*//"; done
done

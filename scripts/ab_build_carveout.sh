for rep in 1 2; do
echo "== bvs"; HESP_LIB=build/ab/bvs.so python scripts/probe_throughput.py C2 100000 2>&1 | tail -1
echo "== nd default-carveout"; HESP_CARVEOUT_BUILD=-1 HESP_LIB=build/ab/nd.so python scripts/probe_throughput.py C2 100000 2>&1 | tail -1
echo "== nd carveout 30"; HESP_CARVEOUT_BUILD=30 HESP_LIB=build/ab/nd.so python scripts/probe_throughput.py C2 100000 2>&1 | tail -1
done
for arm in "bvs::" "nd:-1:" "nd:30:"; do IFS=: read lib cv x <<< "$arm"
env ${cv:+HESP_CARVEOUT_BUILD=$cv} HESP_LIB=build/ab/$lib.so HESP_CHUNK=32768 ncu --metrics l1tex__t_sector_hit_rate.pct,launch__shared_mem_config_size,gpu__time_duration.sum --clock-control none -k regex:"build_kernel" -s 1 -c 1 --csv python scripts/probe_throughput.py C2 32768 2>/dev/null | grep -E "build_kernel" | awk -v a="$lib$cv" -F'","' '{print a, $(NF-2), $NF}'
done

#!/bin/bash
# L1/SMEM carveout A/B per kernel (percent of the maximum shared memory), ncu L1 hit per arm
P=${1:-C2}; N=${2:-100000}
for rep in 1 2; do
  echo "== default"; python scripts/probe_throughput.py $P $N 2>&1 | tail -1
  for c in 22 25 30; do echo "== sim carveout $c"; HESP_CARVEOUT_SIM=$c python scripts/probe_throughput.py $P $N 2>&1 | tail -1; done
done
for c in 22 25; do
  HESP_CARVEOUT_SIM=$c HESP_CHUNK=32768 timeout 600 ncu --metrics l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,launch__shared_mem_config_size,sm__warps_active.avg.per_cycle_active --clock-control none -k regex:"sim_kernel" -s 1 -c 1 --csv python scripts/probe_throughput.py C2 32768 2>/dev/null | grep -E "sim_kernel" > gpurun_out/ncu_carveout_sim_$c.csv
done

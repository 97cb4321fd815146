#!/bin/bash
# SMEM-staging experiment: the lean loop's valid-time table in
# shared memory (HESP_VSTAGE bytes per warp) at fewer resident CTAs, vs the
# default (8 CTAs/SM, table in the slot).
P=${1:-C2}; N=${2:-100000}
for rep in 1 2; do
  echo "== default (8 CTAs/SM)"; python scripts/probe_throughput.py $P $N 2>&1 | tail -1
  echo "== 6 CTAs/SM, table in the slot"; HESP_SIM_CTAS=6 python scripts/probe_throughput.py $P $N 2>&1 | tail -1
  echo "== 6 CTAs/SM, table in SMEM (7 KB/warp)"; HESP_SIM_CTAS=6 HESP_VSTAGE=7168 python scripts/probe_throughput.py $P $N 2>&1 | tail -1
  echo "== 4 CTAs/SM, table in SMEM (12 KB/warp)"; HESP_SIM_CTAS=4 HESP_VSTAGE=12288 python scripts/probe_throughput.py $P $N 2>&1 | tail -1
done

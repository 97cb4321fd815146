#!/bin/bash
# A/B of resident CTAs per SM (HESP_SIM_CTAS / HESP_BUILD_CTAS) on one box.
P=${1:-C2}; N=${2:-100000}
for rep in 1 2; do
  for sc in 8 6 4; do echo "== sim $sc"; HESP_SIM_CTAS=$sc python scripts/probe_throughput.py $P $N 2>&1 | tail -1; done
  for bc in 12 8; do echo "== build $bc"; HESP_BUILD_CTAS=$bc python scripts/probe_throughput.py $P $N 2>&1 | tail -1; done
done

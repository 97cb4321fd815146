#!/bin/bash
# TaskGraph drop-in at volume: N random reference graphs per preset through the C++ bridge
N=${1:-300}
for pr in c2 c3 sect_cpugpu evict_wb merge_sect; do
  args=$(python -c "
from paper_1602_05510_b200.configs import PARITY, harness_args
from paper_1602_05510_b200.engine import FIXTURES
print(' '.join(harness_args(PARITY['$pr'][0], FIXTURES)))")
  echo "== $pr"; timeout 900 oracle/_ref/bridge_check $args --graphs $N | tail -3
done

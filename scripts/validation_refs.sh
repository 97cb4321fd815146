#!/bin/bash
# Reference records for a large one-off parity validation (not committed: build/validation/).
# usage: scripts/validation_refs.sh   (needs oracle/_ref/ref_harness, i.e. /root/reference)
set -e
mkdir -p build/validation
run() {  # preset first count
  args=$(python -c "
from paper_1602_05510_b200.configs import PARITY, CONFIGS, harness_args
from paper_1602_05510_b200.engine import FIXTURES
p = CONFIGS.get('$1') or PARITY['$1'][0]
print(' '.join(harness_args(p, FIXTURES)))")
  oracle/_ref/ref_harness $args --first $2 --count $3 --threads $(nproc) --out build/validation/$1_$2_$3.bin
}
run C2 1000000 100000
run C4 1000 600
run merge_sect 10000 20000
run C3 1000000 50000

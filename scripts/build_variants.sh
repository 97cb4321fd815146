#!/bin/bash
# Build engine library variants for an A/B run: scripts/build_variants.sh name "-DFLAG=.." ...
# (outputs build/ab/<name>.so; build/ is git-ignored but travels with gpurun)
mkdir -p build/ab
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  python - "$name" "$flags" <<'PY' &
import sys, subprocess
sys.path.insert(0, '.')
from paper_1602_05510_b200.build import nvcc_command
name, flags = sys.argv[1], sys.argv[2]
cmd = nvcc_command(out=f"build/ab/{name}.so")
cmd[1:1] = flags.split()
subprocess.run(cmd, check=True)
PY
done
wait
ls -la build/ab

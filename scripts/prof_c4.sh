#!/bin/bash
# C4 evidence: bench line + per-kernel counters + one full capture of each kernel.
TAG=${1:-r10}
mkdir -p gpurun_out
timeout 600 python bench.py --config C4 --batch 50000 --steps 3 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err
HESP_CHUNK=8192 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"build_kernel|sim_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_c4_$TAG -f python scripts/probe_throughput.py C4 8192 > gpurun_out/prof_c4_$TAG.log 2>&1
ls -la gpurun_out

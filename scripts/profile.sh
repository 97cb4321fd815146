#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the dominant kernel; run under gpurun.
# usage: scripts/profile.sh <tag> [batch]
set -x
TAG=${1:-r01}; BATCH=${2:-100000}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --batch $BATCH --no-cpu-baseline > gpurun_out/launches_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG -f \
    python bench.py --steps 1 --warmup 1 --batch $BATCH --no-cpu-baseline > gpurun_out/prof_bench_$TAG.log 2>&1

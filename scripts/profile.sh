#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the engine's kernels; run under gpurun.
# usage: scripts/profile.sh <tag>
TAG=${1:-r03}
mkdir -p gpurun_out
# 1) clean bench line (not under a profiler)
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
# 2) launch list of the same command (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# 3) DRAM traffic of one bench step (build + sim kernels of each chunk)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum \
    --clock-control none --csv -k regex:"build_kernel|sim_kernel" -s 2 -c 4 --log-file gpurun_out/traffic_$TAG.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# 4) one full capture of each kernel (a 32k chunk keeps ~40 replays short)
HESP_CHUNK=32768 ncu --set full --import-source on --clock-control none -k regex:"build_kernel|sim_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG -f python scripts/probe_throughput.py C2 32768 > /dev/null 2>&1
ls -la gpurun_out

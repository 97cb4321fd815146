#!/bin/bash
# the A/B of scripts/ab_vstage.sh plus one ncu capture of sim_kernel per arm
bash scripts/ab_vstage.sh C2 100000 > gpurun_out/ab_vstage_c2.txt 2>&1
for arm in "default::" "ctas6:6:" "vstage6:6:7168"; do
  IFS=: read name ctas vst <<< "$arm"
  env ${ctas:+HESP_SIM_CTAS=$ctas} ${vst:+HESP_VSTAGE=$vst} HESP_CHUNK=32768 timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section SchedulerStats --section WarpStateStats --section Occupancy --section LaunchStats --metrics smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sim_kernel -s 1 -c 1 --csv --page details python scripts/probe_throughput.py C2 32768 > gpurun_out/ncu_vstage_$name.csv 2>/dev/null
done
ls -la gpurun_out/*vstage*

# Source-level ncu captures of build_kernel and sim_kernel (one 32k-candidate C2 chunk each).
TAG=$1
HESP_CHUNK=32768 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"build_kernel|sim_kernel" -c 2 \
    -o gpurun_out/prof_$TAG -f python scripts/probe_throughput.py C2 32768 > gpurun_out/prof_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k build_kernel > gpurun_out/srcb_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k sim_kernel > gpurun_out/srcs_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
python scripts/ncu_hot.py gpurun_out/srcb_$TAG.csv 32768 80 > gpurun_out/hotb_$TAG.txt 2>&1
python scripts/ncu_hot.py gpurun_out/srcs_$TAG.csv 32768 80 > gpurun_out/hots_$TAG.txt 2>&1

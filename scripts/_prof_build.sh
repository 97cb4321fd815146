LIB=$1; TAG=$2
HESP_LIB=$LIB HESP_CHUNK=32768 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"build_kernel" -s 1 -c 1 \
    -o gpurun_out/profb_$TAG -f python scripts/probe_throughput.py C2 32768 > gpurun_out/profb_$TAG.log 2>&1
ncu -i gpurun_out/profb_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k build_kernel > gpurun_out/srcb_$TAG.csv 2>/dev/null
ncu -i gpurun_out/profb_$TAG.ncu-rep --page raw --csv > gpurun_out/rawb_$TAG.csv 2>/dev/null

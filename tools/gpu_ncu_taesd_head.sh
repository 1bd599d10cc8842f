cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:conv3x3_c64_u8|conv3x3_rgb8' -c 4 -o gpurun_out/ncu_taesd_head python tools/taesd_prof.py 1 > gpurun_out/ncu_taesd_head.log 2>&1
ncu -i gpurun_out/ncu_taesd_head.ncu-rep > gpurun_out/ncu_taesd_head.txt 2>&1
grep -E "conv3x3|Duration|Throughput|Busy|Warp Cycles|Eligible|Occupancy|Stall|No Eligible|Registers" gpurun_out/ncu_taesd_head.txt | head -60

cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --cache-control none --clock-control none --csv --log-file gpurun_out/unet_launches.csv python tools/prof_unet.py 4 2 > gpurun_out/unet_launches.log 2>&1
NCU="ncu --set full --clock-control none --cache-control none --import-source on"
timeout 300 $NCU -k regex:gn_stats -s 30 -c 1 -o gpurun_out/ncu_gnstats python tools/prof_unet.py 4 1 > /dev/null 2>&1
timeout 300 $NCU -k regex:gn_apply -s 30 -c 1 -o gpurun_out/ncu_gnapply python tools/prof_unet.py 4 1 > /dev/null 2>&1

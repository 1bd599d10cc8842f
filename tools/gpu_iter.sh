cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
M="--clock-control none --cache-control none"
timeout 300 python tools/attn_probe.py > gpurun_out/attn_probe.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum $M --profile-from-start off --csv --log-file gpurun_out/unet_traffic_r8.csv python tools/prof_unet.py 8 3 > gpurun_out/ncu_traffic_r8.log 2>&1
python tools/ncu_traffic.py gpurun_out/unet_traffic_r8.csv gpurun_out/unet_traffic_r8.json "UNet forward, 8 rows (cfg4 denoiser launch)" 8 > gpurun_out/unet_traffic_r8.txt

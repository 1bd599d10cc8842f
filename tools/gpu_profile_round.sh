#!/bin/bash
# Round profile artefacts: bench launch list (cfg1), DRAM traffic of one UNet forward
# (4 rows, the cfg1 denoiser launch), ncu --set full of the top conv and attention kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
M="--clock-control none --cache-control none"
timeout 900 ncu --metrics gpu__time_duration.sum $M --profile-from-start off --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --profile-window > gpurun_out/ncu_cfg1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum $M --profile-from-start off --csv --log-file gpurun_out/unet_traffic.csv python tools/prof_unet.py 4 3 > gpurun_out/ncu_traffic.log 2>&1
python tools/ncu_traffic.py gpurun_out/unet_traffic.csv gpurun_out/unet_traffic.json "UNet forward, 4 rows (cfg1 denoiser launch)" 4 > gpurun_out/unet_traffic.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum $M --profile-from-start off --csv --log-file gpurun_out/unet_traffic_r8.csv python tools/prof_unet.py 8 3 > gpurun_out/ncu_traffic_r8.log 2>&1
python tools/ncu_traffic.py gpurun_out/unet_traffic_r8.csv gpurun_out/unet_traffic_r8.json "UNet forward, 8 rows (cfg4 denoiser launch)" 8 > gpurun_out/unet_traffic_r8.txt
NCU="ncu --set full $M --import-source on"
timeout 600 $NCU -k regex:gemm_tc -s 12 -c 1 --profile-from-start off -o gpurun_out/ncu_full_gemm python tools/prof_unet.py 4 2 > gpurun_out/ncu_full_gemm.log 2>&1
timeout 600 $NCU -k regex:attn -s 0 -c 1 --profile-from-start off -o gpurun_out/ncu_full_attn python tools/prof_unet.py 4 2 > gpurun_out/ncu_full_attn.log 2>&1
ls -la gpurun_out

#!/bin/bash
# Per-op UNet profile, GEMM vs cuBLAS, GN-fuse A/B, ncu --set full of the top kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/prof_ops.py 4 5 > gpurun_out/prof_ops_r4.txt 2>&1
timeout 300 python tools/prof_ops.py 8 5 > gpurun_out/prof_ops_r8.txt 2>&1
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1
SDX_GN_FUSE=1 timeout 300 python tools/prof_ops.py 4 5 > gpurun_out/prof_ops_r4_gnfuse.txt 2>&1
SDX_GN_FUSE=1 timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_gnfuse.json 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:gemm_tc_kernel<160, 5, 2>' -s 1 -c 1 -o gpurun_out/ncu_conv160 python tools/prof_unet.py 4 1 > gpurun_out/ncu_conv160.log 2>&1
timeout 600 $NCU -k 'regex:gemm_tc_kernel<256, 4, 0>' -s 4 -c 1 -o gpurun_out/ncu_lin256 python tools/prof_unet.py 4 1 > gpurun_out/ncu_lin256.log 2>&1
timeout 600 $NCU -k 'regex:attn_kernel' -s 0 -c 1 -o gpurun_out/ncu_attn python tools/prof_unet.py 4 1 > gpurun_out/ncu_attn.log 2>&1
timeout 600 $NCU -k 'regex:gn_stats_kernel' -s 2 -c 1 -o gpurun_out/ncu_gnstats python tools/prof_unet.py 4 1 > gpurun_out/ncu_gnstats.log 2>&1
timeout 600 $NCU -k 'regex:splitk_reduce' -s 2 -c 1 -o gpurun_out/ncu_splitk python tools/prof_unet.py 4 1 > gpurun_out/ncu_splitk.log 2>&1
timeout 900 $NCU -k 'regex:gemm_tc_kernel<64, 6, 2>' -s 10 -c 1 -o gpurun_out/ncu_taesd64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_taesd64.log 2>&1
ls -la gpurun_out

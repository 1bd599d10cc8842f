cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:gemm_tc_kernel' -s 2 -c 1 -o gpurun_out/ncu_lin320 python tools/one_gemm.py gemm 16384 320 320 1 > gpurun_out/ncu_lin320.log 2>&1
timeout 600 $NCU -k 'regex:gemm_tc_kernel' -s 2 -c 1 -o gpurun_out/ncu_lin1280 python tools/one_gemm.py gemm 1024 1280 1280 1 > gpurun_out/ncu_lin1280.log 2>&1
timeout 600 $NCU -k 'regex:gemm_tc_kernel' -s 2 -c 1 -o gpurun_out/ncu_conv320 python tools/one_gemm.py conv 4 64 320 320 > gpurun_out/ncu_conv320.log 2>&1
ls gpurun_out/*.ncu-rep

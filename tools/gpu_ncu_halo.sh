# ncu --set full of the TAESD halo conv (8 x 512^2, 64 -> 64) with source-level stall sampling
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:gemm_tc_kernel' -s 2 -c 1 -o gpurun_out/ncu_halo python tools/one_gemm.py conv 8 512 64 64 > gpurun_out/ncu_halo.log 2>&1
ncu -i gpurun_out/ncu_halo.ncu-rep > gpurun_out/ncu_halo.txt 2>&1
ncu -i gpurun_out/ncu_halo.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_halo_sass.csv 2>/dev/null
grep -E "gemm_tc|Duration|Throughput|Pipe|pipe|Busy|Eligible|Shared" gpurun_out/ncu_halo.txt | head -40
python tools/ncu_sass_hot.py gpurun_out/ncu_halo_sass.csv 25

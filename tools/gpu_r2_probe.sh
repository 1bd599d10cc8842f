# GEMM/conv pipeline probes (full vs TMA-only vs MMA-only) + ncu full of the 64^2 320->320 conv
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:gemm_tc_kernel' -s 2 -c 1 -o gpurun_out/ncu_conv320 python tools/one_gemm.py conv 4 64 320 320 > gpurun_out/ncu_conv320.log 2>&1
ncu -i gpurun_out/ncu_conv320.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_conv320_sass.csv 2>/dev/null
ncu -i gpurun_out/ncu_conv320.ncu-rep > gpurun_out/ncu_conv320_details.txt 2>/dev/null
cat gpurun_out/gemm_probe.txt
python tools/ncu_sass_hot.py gpurun_out/ncu_conv320_sass.csv 30
grep -E "Duration|Throughput|Pipe|pipe" gpurun_out/ncu_conv320_details.txt | head -30

# ncu --set full of the GroupNorm cluster kernel at the UNet's 64^2 x 320 shape (4 images)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NCU -k 'regex:gn_cluster' -s 3 -c 1 -o gpurun_out/ncu_gn python tools/gn_bench.py 4 > gpurun_out/ncu_gn.log 2>&1
ncu -i gpurun_out/ncu_gn.ncu-rep > gpurun_out/ncu_gn.txt 2>&1
ncu -i gpurun_out/ncu_gn.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_gn_sass.csv 2>/dev/null
grep -E "gn_cluster|Duration|Elapsed Cycles|SM Active|Throughput|Busy|Eligible|Occupancy" gpurun_out/ncu_gn.txt | head -30
python tools/ncu_sass_hot.py gpurun_out/ncu_gn_sass.csv 20

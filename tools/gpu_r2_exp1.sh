# microbenchmarks + L2 weight-hint A/B on the whole-forward time
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for b in ubench_mma ubench_launch ubench_tma ubench_tma_lat; do echo "== $b"; timeout 60 tools/ubench/_bin/$b; done > gpurun_out/ubench.txt 2>&1
bash tools/ab_env.sh "SDX_WHINT=0" 4 > gpurun_out/ab_whint4.txt 2>&1
bash tools/ab_env.sh "SDX_WHINT=0" 8 > gpurun_out/ab_whint8.txt 2>&1
cat gpurun_out/ubench.txt gpurun_out/ab_whint4.txt gpurun_out/ab_whint8.txt

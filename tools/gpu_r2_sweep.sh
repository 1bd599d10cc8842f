# TAESD per-op profile + full GEMM tiling sweep (rows 2, 4, 8) with the records for fit_tiling.py
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/taesd_prof.py 1 8 > gpurun_out/taesd_prof.txt 2>&1
SDX_SWEEP_JSON=gpurun_out/sweep_all.json timeout 1500 python tools/gemm_sweep.py 2 4 8 > gpurun_out/gemm_sweep.txt 2>&1
cat gpurun_out/taesd_prof.txt; tail -3 gpurun_out/gemm_sweep.txt

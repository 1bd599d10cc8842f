# weight prefetch before the PDL wait: kernel/UNet/TAESD parity + whole-forward A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_unet_gpu.py tests/test_taesd_gpu.py -q -x > gpurun_out/t_kern.txt 2>&1; echo "rc=$?" >> gpurun_out/t_kern.txt
tail -3 gpurun_out/t_kern.txt
bash tools/ab_env.sh "SDX_WPREFETCH=0" 4 > gpurun_out/ab_wpre4.txt 2>&1
bash tools/ab_env.sh "SDX_WPREFETCH=0" 8 > gpurun_out/ab_wpre8.txt 2>&1
timeout 120 python tools/taesd_prof.py 1 8 > gpurun_out/taesd_prof2.txt 2>&1
SDX_WPREFETCH=0 timeout 120 python tools/taesd_prof.py 1 8 > gpurun_out/taesd_prof2_off.txt 2>&1
timeout 60 tools/ubench/_bin/ubench_pipes > gpurun_out/ubench_pipes.txt 2>&1
cat gpurun_out/ab_wpre4.txt gpurun_out/ab_wpre8.txt; grep "===" gpurun_out/taesd_prof2.txt gpurun_out/taesd_prof2_off.txt; cat gpurun_out/ubench_pipes.txt

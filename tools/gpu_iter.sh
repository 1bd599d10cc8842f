cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
rm -f gpurun_out/attn_poly.txt
for P in 0 2 3 4; do
  echo "POLY=$P" >> gpurun_out/attn_poly.txt
  SDX_ATTN_POLY=$P timeout 300 python tools/attn_probe.py 2>&1 | cut -c1-80 >> gpurun_out/attn_poly.txt
done
SDX_ATTN_POLY=4 timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_unet_gpu.py -m gpu -x -q -k "attention or unet" > gpurun_out/t_poly.txt 2>&1

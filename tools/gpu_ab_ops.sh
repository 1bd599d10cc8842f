# per-op profile + whole-forward time of several builds on one box: bash tools/gpu_ab_ops.sh base new [...]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
vs="${@:-base new}"
for v in $vs; do
  cp ab/lib_$v.so paper_2312_12491_b200/libstagger_b200.so
  timeout 300 python tools/prof_ops.py 4 > gpurun_out/ops_$v.txt 2>&1
  timeout 100 python tools/unet_time.py 4 8 >> gpurun_out/ops_$v.txt 2>&1
done
cp ab/lib_new.so paper_2312_12491_b200/libstagger_b200.so
for v in $vs; do echo "== $v"; sed -n 1p gpurun_out/ops_$v.txt; sed -n 4,7p gpurun_out/ops_$v.txt; tail -2 gpurun_out/ops_$v.txt; done

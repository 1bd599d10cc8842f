cd "${GRAFT_REPO_ROOT:-.}"
B1="timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python tools/bench_line.py"
for i in 1 2; do
  cp ab/lib_new.so paper_2312_12491_b200/libstagger_b200.so
  echo "new: $(eval $B1)"
  echo "new WPREFETCH=0: $(SDX_WPREFETCH=0 eval $B1)"
  echo "new unet_time: $(timeout 100 python tools/unet_time.py 4)"
  echo "new unet_time WPREFETCH=0: $(SDX_WPREFETCH=0 timeout 100 python tools/unet_time.py 4)"
  cp ab/lib_base.so paper_2312_12491_b200/libstagger_b200.so
  echo "base unet_time: $(timeout 100 python tools/unet_time.py 4)"
done
cp ab/lib_new.so paper_2312_12491_b200/libstagger_b200.so

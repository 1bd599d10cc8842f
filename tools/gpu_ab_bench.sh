# same-box A/B of ab/lib_base.so vs ab/lib_new.so on the cfg1 and cfg4 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
B1="timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python tools/bench_line.py"
B4="timeout 300 python bench.py --streams 8 --n-steps 1 --guidance self_negative --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python tools/bench_line.py"
echo "cfg1"; bash tools/ab_lib.sh "$B1" 2
echo "cfg4"; bash tools/ab_lib.sh "$B4" 2

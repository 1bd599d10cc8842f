# Same-box A/B of two builds of libstagger_b200.so (ab/lib_base.so vs ab/lib_new.so),
# alternating: bash tools/ab_lib.sh "<command printing one timing line>" [repeats]
cd "${GRAFT_REPO_ROOT:-.}"
L=paper_2312_12491_b200/libstagger_b200.so
for i in $(seq 1 ${2:-2}); do
  for v in base new; do
    cp ab/lib_$v.so $L
    echo "== $v: $(eval "$1" 2>&1 | tr '\n' ' ' | cut -c1-400)"
  done
done
cp ab/lib_new.so $L

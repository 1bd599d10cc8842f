cd "${GRAFT_REPO_ROOT:-.}"
for envv in "X=0" "SDX_GN_CLUSTER_MAX=0" "SDX_GN_CLUSTER_SIZE=8"; do
  echo "== $envv: $(env $envv timeout 100 python tools/unet_time.py 4 | tr '\n' ' ')"
  env $envv timeout 200 python tools/prof_ops.py 4 2>&1 | grep -E "^  groupnorm|groupnorm HW=4096 C=320|groupnorm HW=64 C=1280 "
done

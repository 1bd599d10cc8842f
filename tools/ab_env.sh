# A/B of an environment switch on the whole-forward time: alternating processes.
#   bash tools/ab_env.sh "SDX_WPREFETCH=0" [rows]
cd "${GRAFT_REPO_ROOT:-.}"
rows=${2:-4}
for i in 1 2 3; do
  echo "A: $(timeout 200 python tools/unet_time.py $rows)"
  echo "B ($1): $(env $1 timeout 200 python tools/unet_time.py $rows)"
done

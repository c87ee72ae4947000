# Sweeps an env var over values: bash scripts/gpu_env_sweep.sh VAR "v1 v2 .." scene scale ... (dev aid)
cd "${GRAFT_REPO_ROOT:-.}"
L=paper_1812_05902_b200/libraybos_gpu.so
V=$1; VALS=$2; shift 2
for r in 1 2; do
  for v in $VALS; do
    env $V=$v python scripts/sweep.py $L "$@" | sed "s/^/$V=$v /"
  done
done

# A/B of an env toggle: bash scripts/gpu_ab.sh VAR "scenes..."  (dev aid)
cd "${GRAFT_REPO_ROOT:-.}"
L=paper_1812_05902_b200/libraybos_gpu.so
V=$1; shift
for r in 1 2; do
  env $V=0 python scripts/sweep.py $L "$@" | sed "s/^/$V=0 /"
  python scripts/sweep.py $L "$@" | sed "s/^/$V=1 /"
done

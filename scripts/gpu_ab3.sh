# A/B/C of three library variants (dev aid): bash scripts/gpu_ab3.sh tagA tagB tagC [rounds]
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
for r in $(seq ${4:-2}); do
  for t in $1 $2 $3; do
    timeout 600 python scripts/sweep.py $V/libraybos_gpu_$t.so tomo 0.1 bos 0.05 optics 0.1 2>/dev/null
  done
done | tee gpurun_out/ab.jsonl

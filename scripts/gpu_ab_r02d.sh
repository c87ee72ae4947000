# A/B of library variants on the field scenes (dev aid): bash scripts/gpu_ab_r02d.sh tagA tagB ...
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for t in "$@"; do
    timeout 900 python scripts/sweep.py $V/libraybos_gpu_$t.so tomo 0.1 bos 0.05 large 0.002 2>/dev/null
  done
done | tee $O/ab_d.jsonl

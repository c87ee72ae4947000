# A/B of library variants on all four scenes (dev aid): bash scripts/gpu_ab_r02c.sh tagA tagB ...
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for t in "$@"; do
    timeout 600 python scripts/sweep.py $V/libraybos_gpu_$t.so piv 1 optics 0.1 tomo 0.1 bos 0.05 2>/dev/null
  done
done | tee $O/ab_c.jsonl

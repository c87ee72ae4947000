# A/B of library variants + split sweep (dev aid)
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  for t in "$@"; do
    timeout 600 python scripts/sweep.py $V/libraybos_gpu_$t.so tomo 0.1 bos 0.05 2>/dev/null
  done
done | tee $O/ab.jsonl
for sp in 4 8 16; do
  RAYBOS_SPLIT=$sp timeout 600 python scripts/sweep.py $V/libraybos_gpu_v0.so tomo 0.1 2>/dev/null | sed "s/^/split=$sp /"
done | tee $O/ab_split.txt

# A/B: field-kernel tile cap 2048 (base) vs 1024 words (more L1 for the cell table) — variant libraries.
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
for rep in 1 2; do
  for t in base t1024; do
    timeout 900 python scripts/sweep.py $V/libraybos_gpu_$t.so tomo 1 bos 1 large 0.1 2>/dev/null | sed "s/^/$rep $t /"
  done
done

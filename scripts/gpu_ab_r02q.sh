# A/B: 256-thread CTAs (3/SM) vs 384-thread CTAs (2/SM, pair mode compiled out) — variant libraries.
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
for rep in 1 2; do
  for t in base b384; do
    timeout 900 python scripts/sweep.py $V/libraybos_gpu_$t.so tomo 1 bos 1 large 0.1 piv 1 optics 1 2>/dev/null | sed "s/^/$rep $t /"
  done
done

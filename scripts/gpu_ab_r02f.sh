# CTA vs warp K1 for tile caps (dev aid)
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
for t in c2k c4k; do
  for k in cta warp; do
    RAYBOS_K1=$k timeout 900 python scripts/sweep.py $V/libraybos_gpu_$t.so tomo 0.1 bos 0.05 large 0.002 2>/dev/null | sed "s/^/$t $k /"
  done
done

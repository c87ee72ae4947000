# cell-table layout A/B (dev aid)
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
O=gpurun_out; mkdir -p $O
for r in 1 2; do
  timeout 900 python scripts/sweep.py $V/libraybos_gpu_t2k.so tomo 0.1 bos 0.05 large 0.002 2>/dev/null | sed 's/^/old /'
  for lay in x z; do
    RAYBOS_CELL_LAYOUT=$lay timeout 900 python scripts/sweep.py $V/libraybos_gpu_z.so tomo 0.1 bos 0.05 large 0.002 2>/dev/null | sed "s/^/layout=$lay /"
  done
done | tee $O/ab_e.txt

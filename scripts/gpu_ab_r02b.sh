# split sweep with the straight pilot + large A/B (dev aid)
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
O=gpurun_out; mkdir -p $O
for sp in 12 16 25 40; do
  RAYBOS_SPLIT=$sp timeout 600 python scripts/sweep.py $V/libraybos_gpu_v4.so bos 0.05 2>/dev/null | sed "s/^/bos split=$sp /"
done | tee $O/ab_split_bos.txt
for sp in 4 6 8 12; do
  RAYBOS_SPLIT=$sp timeout 600 python scripts/sweep.py $V/libraybos_gpu_v4.so tomo 0.1 2>/dev/null | sed "s/^/tomo split=$sp /"
done | tee $O/ab_split_tomo.txt
for t in v3 v4; do
  timeout 900 python scripts/sweep.py $V/libraybos_gpu_$t.so large 0.005 2>/dev/null
done | tee $O/ab_large.txt

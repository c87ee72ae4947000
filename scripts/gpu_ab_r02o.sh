# No-medium tile cap (RB_TILE_CAP) for the aberrated optics scene and piv (variant libraries).
cd "${GRAFT_REPO_ROOT:-.}"
V=paper_1812_05902_b200/_variants
for rep in 1 2; do
  for t in 6144 12288 16384; do
    timeout 900 python scripts/sweep.py $V/libraybos_gpu_nm$t.so optics 1 piv 1 2>/dev/null | sed "s/^/$rep nm$t /"
  done
done
# value-vs-kernel gap of the tomo bench with split 1 vs 8
for sp in 1 8 1 8; do
  RAYBOS_SPLIT=$sp timeout 900 python bench.py --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline > gpurun_out/bench_o.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_o.json').read().strip().splitlines()[-1])
print('split $sp ms_per_step %.2f kernel %.2f e2e %.2f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['ms_per_step']))"
done

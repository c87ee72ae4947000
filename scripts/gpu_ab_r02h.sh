# Emitter-split sweep for the no-medium scenes (RAYBOS_SPLIT), full-scale piv / optics.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for sc in piv optics; do
  for sp in auto 1 2 3 4 6; do
    if [ $sp = auto ]; then unset RAYBOS_SPLIT; else export RAYBOS_SPLIT=$sp; fi
    timeout 600 python bench.py --scene $sc --steps 10 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_h.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/bench_h.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$rep $sc split $sp value %.4g step %.4f kernel %.4f frac %.4f chk %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum']))"
  done
done
done
unset RAYBOS_SPLIT

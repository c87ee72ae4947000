# Emitter-split sweep with the band-order patches (stride 1) in the field kernels.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for cfg in "tomo 1" "tomo 2" "bos 3" "bos 4" "bos 6" "large 40" "large 5"; do
  set -- $cfg
  if [ $2 = auto ]; then unset RAYBOS_SPLIT; else export RAYBOS_SPLIT=$2; fi
  timeout 1200 python bench.py --scene $1 --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_n.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/bench_n.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$rep $1 split $2 value %.4g kernel %.2f frac %.4f chk %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum']))"
done
done
unset RAYBOS_SPLIT

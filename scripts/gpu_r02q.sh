cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python scripts/warp_k1_check.py > $O/warp_check.log 2>&1; echo "check rc=$?"; tail -4 $O/warp_check.log
for sc in bos large tomo; do
  for k in cta auto; do
    RAYBOS_K1=$( [ $k = auto ] && echo "" || echo $k ) timeout 1200 python bench.py --scene $sc --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_q_${sc}_$k.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/bench_q_${sc}_$k.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$sc $k value %.4g kernel %.2f frac %.4f chk %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum']))"
  done
done

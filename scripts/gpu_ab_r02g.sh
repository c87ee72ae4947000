# A/B: render_emitters vs render_warps (global queue) vs render_warps (CTA pool), full-scale scenes.
# (the CTA-pool variant, RAYBOS_K1=wpool, was measured here and removed: tomo +1% over warp, still -9% vs cta)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_k1_variants.py -q -x > $O/g_variants.log 2>&1; echo "variants rc=$?"; tail -2 $O/g_variants.log
for rep in 1 2; do
for sc in tomo bos large; do
  for k in cta warp wpool; do
    RAYBOS_K1=$k timeout 1200 python bench.py --scene $sc --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_g_${sc}_$k.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/bench_g_${sc}_$k.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$rep $sc $k value %.4g kernel %.2f frac %.4f chk %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum']))"
  done
done
done

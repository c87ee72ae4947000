# A/B (one box, 3 rounds): render_emitters with patch stride 1 vs render_warps
# items in band order (warp) vs in render_emitters' coprime slot order (wslot).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
for sc in tomo bos large; do
  for k in cta1 warp wslot; do
    unset RAYBOS_PATCH_STRIDE
    if [ $k = cta1 ]; then export RAYBOS_PATCH_STRIDE=1; fi
    RAYBOS_K1=${k%1} timeout 1200 python bench.py --scene $sc --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_l_${sc}_$k.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/bench_l_${sc}_$k.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$rep $sc $k value %.4g kernel %.2f frac %.4f chk %s %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum'], r['kernel']))"
  done
done
done

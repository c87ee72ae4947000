# A/B: render_emitters vs render_warps with pupil-neighbour items, full-scale scenes.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_k1_variants.py -q -x > $O/i_variants.log 2>&1; echo "variants rc=$?"; tail -2 $O/i_variants.log
for rep in 1 2; do
for sc in tomo bos large; do
  for k in cta warp; do
    RAYBOS_K1=$k timeout 1200 python bench.py --scene $sc --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_i_${sc}_$k.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/bench_i_${sc}_$k.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$rep $sc $k value %.4g kernel %.2f frac %.4f chk %s %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum'], r['kernel']))"
  done
done
done
F="python scripts/run_scene.py tomo 0.02"
RAYBOS_K1=warp $F > $O/i_plain.log 2>&1 && RAYBOS_K1=warp ncu --set full --clock-control none --import-source on -k regex:render_ -s 1 -c 1 -o $O/profi_warp $F > $O/i_ncu.log 2>&1; echo "ncu rc=$?"

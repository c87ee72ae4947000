# A/B: rows per pupil band in the field kernels (RAYBOS_BAND_ROWS 4 / 8 / 16), one box.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
RAYBOS_BAND_ROWS=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_k1_variants.py -q -x > $O/p_tests16.log 2>&1; echo "tests(band 16) rc=$?"; tail -1 $O/p_tests16.log
for rep in 1 2; do
for sc in tomo bos large; do
  for b in 4 8 16; do
    RAYBOS_BAND_ROWS=$b timeout 1200 python bench.py --scene $sc --steps 3 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/bench_p.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/bench_p.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$rep $sc band $b value %.4g kernel %.2f frac %.4f chk %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']['fixed_point_sum']))"
  done
done
done

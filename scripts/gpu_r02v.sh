# Final driver-equivalent pass of round 2 (band-order patches, 8-row bands, re-tuned split) + ncu of the field scenes.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/v_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/v_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/v_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/v_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/v_smoke.log
timeout 1200 python bench.py > $O/v_bench.json 2> $O/v_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/v_bench.json').read().strip().splitlines()[-1])
rows=[('tomo',d)]+list(d['configs'].items())
for k,v in rows:
    r=v['roofline']; print(k, '%.4g'%v['value'], '%.4g'%v['e2e']['value'], round(r['frac'],4), v['image_checksum']['fixed_point_sum'], r['kernel'])
PY
timeout 900 python bench.py --impl reference > $O/v_bench_ref.json 2> $O/v_bench_ref.err; echo "ref rc=$?"
for sc in "tomo 1" "bos 1" "large 0.005"; do
  set -- $sc
  CMD="python scripts/run_scene.py $1 $2"
  timeout 900 $CMD > $O/plainv_$1.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o $O/prof02b_$1 $CMD > $O/ncu02v_$1.log 2>&1
  echo "ncu $1 rc=$?"
done

cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_j.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_j.log
timeout 900 python scripts/bench_parity.py > $O/parity_j.jsonl 2>&1; echo "parity rc=$?"; cut -c1-250 $O/parity_j.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 --no-extra-configs --no-cpu-baseline > $O/bench_j.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_j.json').read().strip().splitlines()[-1]); r=d['roofline']
print('tomo value %.4g ms %.2f kernel %.2f frac %.4f chk %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['image_checksum']))"

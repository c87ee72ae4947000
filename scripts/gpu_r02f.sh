cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_f.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_f.log
timeout 900 python scripts/bench_parity.py > $O/parity_f.jsonl 2>&1; echo "parity rc=$?"; cut -c1-400 $O/parity_f.jsonl
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_f.json 2> $O/bench_f.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_f.json').read().strip().splitlines()[-1])
def show(n,e):
    r=e['roofline']; c=e.get('cpu_baseline') or {}
    print(f"{n:7s} value {e['value']:.4e} e2e {e['e2e']['value']:.4e} ms/step {e['ms_per_step']:.3f} kernel {r['kernel_ms']:.3f} frac {r['frac']:.4f} {r['bound']} cpu {c.get('value')} chk {e['image_checksum']['identical_to_warmup']}")
show('tomo', d)
for k,e in d['configs'].items(): show(k,e)
PY

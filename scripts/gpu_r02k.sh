# round-2 driver-equivalent pass: GPU tests, smoke, the default bench (all configs), the reference arm
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_k.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke_k.log
timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_k.json 2> $O/bench_k.err; echo "bench rc=$?"
timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_k_ref.json 2> $O/bench_k_ref.err; echo "ref rc=$?"; cat $O/bench_k_ref.json | head -c 1500
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_k.json').read().strip().splitlines()[-1])
def show(n,e):
    r=e['roofline']; c=e.get('cpu_baseline') or {}
    print(f"{n:7s} value {e['value']:.4e} e2e {e['e2e']['value']:.4e} ms/step {e['ms_per_step']:.3f} kernel {r['kernel_ms']:.3f} frac {r['frac']:.4f} {r['bound']} cpu {c.get('value')} chk {e['image_checksum']['identical_to_warmup']}")
show('tomo', d)
for k,e in d['configs'].items(): show(k,e)
print(d['clocks'])
PY

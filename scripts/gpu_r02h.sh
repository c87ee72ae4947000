cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1200 python scripts/bos_theory_check.py gpu profiles/r02_bos_theory_reference_stats.npz $O/bos_theory.json > $O/bos_theory.log 2>&1; echo "bos theory rc=$?"; tail -40 $O/bos_theory.log
timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_h.json 2> $O/bench_h.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_h.json').read().strip().splitlines()[-1])
def show(n,e):
    r=e['roofline']; c=e.get('cpu_baseline') or {}
    print(f"{n:7s} value {e['value']:.4e} e2e {e['e2e']['value']:.4e} ms/step {e['ms_per_step']:.3f} kernel {r['kernel_ms']:.3f} frac {r['frac']:.4f} {r['bound']} traffic {r.get('traffic')} cpu {c.get('value')} chk {e['image_checksum']['identical_to_warmup']}")
show('tomo', d)
for k,e in d['configs'].items(): show(k,e)
print(d['clocks'])
PY

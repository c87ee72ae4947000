cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_host_api.py tests/test_gpu_multi.py tests/test_gpu_parity.py -x -q > $O/pytest_l.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_l.log
for sc in piv optics tomo; do
  timeout 900 python bench.py --scene $sc --steps 5 --warmup 3 --no-extra-configs --no-cpu-baseline > $O/bench_l_$sc.json 2>/dev/null; echo "bench $sc rc=$?"
  python -c "
import json; d=json.loads(open('$O/bench_l_$sc.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$sc value %.4g ms %.3f e2e %.4g e2e_ms %.3f kernel %.3f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], r['kernel_ms']))"
done

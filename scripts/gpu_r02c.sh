# round 2: full GPU tests after the plan cache, then per-config bench lines and
# an ncu instruction count for the no-medium scenes
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_c.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_c.log
for sc in tomo piv optics bos; do
  timeout 900 python bench.py --scene $sc --steps 5 --warmup 3 --no-extra-configs --no-cpu-baseline > $O/bench_c_$sc.json 2>/dev/null; echo "bench $sc rc=$?"
  python -c "
import json,sys; d=json.loads(open('$O/bench_c_$sc.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$sc', 'value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], 'kernel_ms %.3f'%r['kernel_ms'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%r['frac'])"
done
python bench.py --scene piv --steps 2 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/ncu_piv_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:render_emitters --clock-control none --csv --log-file $O/ncu_nomedium_inst.csv python bench.py --scene piv --steps 2 --warmup 3 --no-extra-configs --no-cpu-baseline --no-e2e > $O/ncu_piv.log 2>&1; echo "ncu rc=$?"

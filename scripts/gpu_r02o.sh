cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_parity.py tests/test_gpu_bench_scenes.py -x -q > $O/pytest_o.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_o.log
timeout 900 python bench.py --scene bos --steps 5 --warmup 3 --no-extra-configs --no-cpu-baseline > $O/bench_o_bos.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('$O/bench_o_bos.json').read().strip().splitlines()[-1]); r=d['roofline']
print('bos value %.4g kernel %.2f frac %.4f chk %s' % (d['value'], r['kernel_ms'], r['frac'], d['image_checksum']))"

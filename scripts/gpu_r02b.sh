# round 2: new fixtures, bench-scene parity with the off-axis optics camera, the acceptance gate
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_scenes.py tests/test_gpu_acceptance.py tests/test_gpu_fp64.py -q -x > $O/pytest_b.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_b.log
cat $O/acceptance_gpu.log

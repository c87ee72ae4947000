cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1200 python scripts/bos_theory_check.py gpu profiles/r02_bos_theory_reference_stats.npz $O/bos_theory.json > $O/bos_theory.log 2>&1; echo "bos theory rc=$?"; grep -A12 "landed_identical" $O/bos_theory.log; tail -3 $O/bos_theory.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > $O/pytest_i.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_i.log

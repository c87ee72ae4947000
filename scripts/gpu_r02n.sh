cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/pytest_n.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_n.log
bash scripts/gpu_prof_r02b.sh

cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_g.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_g.log
timeout 900 python scripts/bench_parity.py > $O/parity_g.jsonl 2>&1; echo "parity rc=$?"; cut -c1-300 $O/parity_g.jsonl
bash scripts/gpu_prof_r02b.sh

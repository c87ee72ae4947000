cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 1200 python bench.py > $O/bench_tomo.json 2> $O/bench_tomo.err; echo "bench rc=$?"; cat $O/bench_tomo.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_tomo.json 2> $O/bench_ref.err; echo "ref rc=$?"; cat $O/bench_ref_tomo.json

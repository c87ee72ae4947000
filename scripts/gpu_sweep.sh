cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for lib in paper_1812_05902_b200/_variants/*.so; do timeout 300 python scripts/sweep.py $lib; done

cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
./oracle/_ref/adapter_parity | grep -o '"check": "[^"]*".*"image_rel_l2": [^,]*'
python scripts/sweep.py paper_1812_05902_b200/libraybos_gpu.so

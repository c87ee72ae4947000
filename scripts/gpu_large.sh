cd "${GRAFT_REPO_ROOT:-.}"
L=paper_1812_05902_b200/libraybos_gpu.so
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
python scripts/sweep.py $L large 0.01
RAYBOS_CELL_TABLE=2 python scripts/sweep.py $L large 0.01

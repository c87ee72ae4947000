cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
nvidia-smi -L > $O/san_smi.txt 2>&1
timeout 300 python scripts/sanitize_k1.py small blob aberration shock_particles > $O/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool ${TOOL:-memcheck} --error-exitcode 7 --print-limit 50 python scripts/sanitize_k1.py small blob aberration shock_particles > $O/san_${TOOL:-memcheck}.log 2>&1
echo "rc=$?"; tail -5 $O/san_plain.log; tail -15 $O/san_${TOOL:-memcheck}.log

cd "${GRAFT_REPO_ROOT:-.}"
CMD="python scripts/run_scene.py large 0.003"
$CMD > gpurun_out/plain_large.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o gpurun_out/prof_large $CMD > gpurun_out/ncu_large.log 2>&1
echo "large rc=$?"; cat gpurun_out/plain_large.log

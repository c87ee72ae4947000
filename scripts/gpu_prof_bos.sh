cd "${GRAFT_REPO_ROOT:-.}"
CMD="python scripts/run_scene.py bos 0.02"
$CMD > gpurun_out/bos_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o gpurun_out/prof_bos $CMD > gpurun_out/ncu_bos.log 2>&1
echo "rc=$?"; cat gpurun_out/bos_plain.log

cd "${GRAFT_REPO_ROOT:-.}"
CMD="python scripts/run_scene.py bos 0.1"
$CMD > gpurun_out/plain_bos4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o gpurun_out/prof4_bos $CMD > gpurun_out/ncu4_bos.log 2>&1
echo "rc=$?"; cat gpurun_out/plain_bos4.log

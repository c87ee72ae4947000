cd "${GRAFT_REPO_ROOT:-.}"
for sc in "tomo 0.1" "bos 0.1"; do
  set -- $sc
  CMD="python scripts/run_scene.py $1 $2"
  $CMD > gpurun_out/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o gpurun_out/prof8_$1 $CMD > gpurun_out/ncu8_$1.log 2>&1
  echo "$1 rc=$?"; cat gpurun_out/plain_$1.log
done

cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/sweep.py paper_1812_05902_b200/libraybos_gpu.so
for sc in "tomo 0.1" "bos 0.1"; do
  set -- $sc
  CMD="python scripts/run_scene.py $1 $2"
  $CMD > gpurun_out/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o gpurun_out/prof3_$1 $CMD > gpurun_out/ncu3_$1.log 2>&1
  echo "$1 rc=$?"; cat gpurun_out/plain_$1.log
done

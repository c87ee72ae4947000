cd "${GRAFT_REPO_ROOT:-.}"
for lib in old w6; do
  if [ $lib = old ]; then export RAYBOS_LIB=$PWD/paper_1812_05902_b200/_variants/libraybos_gpu_old.so; else export RAYBOS_LIB=$PWD/paper_1812_05902_b200/libraybos_gpu.so; fi
  CMD="python scripts/run_scene.py optics 0.1"
  $CMD > gpurun_out/plain_optics_$lib.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o gpurun_out/prof_optics_$lib $CMD > gpurun_out/ncu_optics_$lib.log 2>&1
  echo "$lib rc=$?"; cat gpurun_out/plain_optics_$lib.log
done

cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for k in warp cta; do
  RAYBOS_K1=$k python scripts/run_scene.py tomo 0.02 > $O/plainw_$k.log 2>&1 && \
  RAYBOS_K1=$k ncu --set full --clock-control none --import-source on -k regex:render_ -s 1 -c 1 -o $O/profw_$k python scripts/run_scene.py tomo 0.02 > $O/ncuw_$k.log 2>&1
  echo "$k rc=$?"; cat $O/plainw_$k.log
done

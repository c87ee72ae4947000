# ncu --set full of K1 on the no-medium scenes and on tomo (round 2)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for sc in "piv 1" "optics 0.1" "tomo 0.02"; do
  set -- $sc
  CMD="python scripts/run_scene.py $1 $2"
  $CMD > $O/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o $O/prof02_$1 $CMD > $O/ncu02_$1.log 2>&1
  echo "$1 rc=$?"; cat $O/plain_$1.log
done

# round 2 ncu captures of K1 at bench scale (large: reduced) + instruction counts
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for sc in "piv 1" "optics 1" "tomo 1" "bos 1" "large 0.005"; do
  set -- $sc
  CMD="python scripts/run_scene.py $1 $2"
  timeout 900 $CMD > $O/plainb_$1.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o $O/prof02b_$1 $CMD > $O/ncu02b_$1.log 2>&1
  echo "$1 rc=$?"; cat $O/plainb_$1.log
done

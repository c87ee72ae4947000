# Full measurement round on one B200 (run via gpurun); outputs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log
timeout 1200 python bench.py > $O/bench_tomo.json 2> $O/bench_tomo.err; echo "bench rc=$?"
for s in bos piv optics; do
  timeout 900 python bench.py --scene $s --steps 3 --warmup 3 > $O/bench_$s.json 2> $O/bench_$s.err; echo "bench $s rc=$?"
done
timeout 1200 python bench.py --scene large --scale 0.125 --steps 3 --warmup 3 > $O/bench_large.json 2> $O/bench_large.err; echo "bench large rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_tomo.json 2> $O/bench_ref.err; echo "ref rc=$?"
L="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$L > $O/launch_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $L > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
F="python scripts/run_scene.py tomo 1.0"
$F > $O/full_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o $O/prof_k1_tomo $F > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
B="python scripts/run_scene.py bos 1.0"
$B > $O/bos_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:render_emitters -s 1 -c 1 -o $O/prof_k1_bos $B > $O/ncu_bos.log 2>&1; echo "ncu bos rc=$?"

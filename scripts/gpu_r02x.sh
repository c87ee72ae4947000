# ncu launch list (gpu__time_duration per launch) of the default tomo bench command, round 2.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
L="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra-configs"
$L > $O/x_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches.csv $L > $O/x_ncu.log 2>&1; echo "ncu launches rc=$?"

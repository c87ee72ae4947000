# Driver-equivalent pass with the warp-level K1 as the default for outside-emitter scenes.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/r_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/r_smoke.log
timeout 1200 python bench.py > $O/r_bench.json 2> $O/r_bench.err; echo "bench rc=$?"; tail -c 600 $O/r_bench.json
timeout 900 python bench.py --impl reference > $O/r_bench_ref.json 2> $O/r_bench_ref.err; echo "ref rc=$?"; tail -c 400 $O/r_bench_ref.json
B="python scripts/run_scene.py bos 1.0"
$B > $O/r_bos_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:render_warps -s 1 -c 1 -o $O/prof_k1w_bos $B > $O/r_ncu_bos.log 2>&1; echo "ncu bos rc=$?"

# round 2: GPU tests + smoke + default bench (all configs) + the N>1 path checks
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
FAKE=$PWD/tests/fake_nccl/libfakenccl.so
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"; tail -c 3000 $O/bench_default.json; tail -3 $O/bench_default.err
RAYBOS_BENCH_BACKEND=gloo RAYBOS_NCCL_LIB=$FAKE timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --scale 0.01 --no-cpu-baseline > $O/dist_ranks.json 2> $O/dist_ranks.err; echo "ranks rc=$?"; cat $O/dist_ranks.json | head -c 1500; grep raybos $O/dist_ranks.err
RAYBOS_BENCH_DEVICES=0,0 RAYBOS_NCCL_LIB=$FAKE timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --scale 0.01 --no-cpu-baseline > $O/dist_inproc.json 2> $O/dist_inproc.err; echo "inproc rc=$?"; head -c 1500 $O/dist_inproc.json; grep raybos $O/dist_inproc.err
timeout 300 python bench.py --steps 2 --warmup 3 --scale 0.01 --no-cpu-baseline --no-extra-configs > $O/single_small.json 2>&1; echo "single rc=$?"; head -c 600 $O/single_small.json

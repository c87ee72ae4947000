# Path check of bench.py's torchrun (N>1) code on a one-GPU box (gloo, ranks share the GPU).
# The fixed-point image checksum at N=2 must equal N=1's; the timings are not measurements.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
A="--scene tomo --scale 0.05 --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 python bench.py $A > $O/dist_n1.json 2> $O/dist_n1.err; echo "n1 rc=$?"
RAYBOS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 $A > $O/dist_n2.json 2> $O/dist_n2.err; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/dist_ref_n2.json 2> $O/dist_ref_n2.err; echo "ref n2 rc=$?"
python - <<'PY'
import json
a = json.loads(open("gpurun_out/dist_n1.json").read().strip().splitlines()[-1])
b = json.loads(open("gpurun_out/dist_n2.json").read().strip().splitlines()[-1])
print("n1", a["image_checksum"], a["value"])
print("n2", b["image_checksum"], b["value"], b["n_gpus"], b["e2e"]["path"])
print("checksums equal:", a["image_checksum"]["fixed_point_sum"] == b["image_checksum"]["fixed_point_sum"])
PY
tail -c 600 $O/dist_ref_n2.json

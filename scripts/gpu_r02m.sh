# torchrun with one rank: the bench's rank mode against the real NCCL (one-rank job)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > $O/torchrun1.json 2> $O/torchrun1.err; echo "torchrun1 rc=$?"
python -c "
import json; d=json.loads(open('$O/torchrun1.json').read().strip().splitlines()[-1]); r=d['roofline']
print('value %.4g e2e %.4g frac %.4f comm %s chk %s' % (d['value'], d['e2e']['value'], r['frac'], d['comm'], d['image_checksum']))"
grep raybos $O/torchrun1.err

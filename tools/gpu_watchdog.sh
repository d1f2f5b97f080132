#!/bin/bash
TAG=${1:-wd1}
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 \
  bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/${TAG}_n2.json 2> gpurun_out/${TAG}_n2.err
echo "n2 rc=$?"; grep '^{' gpurun_out/${TAG}_n2.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], str(d.get('summa_3d'))[:200])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 \
  bench.py --gpus 2 --steps 3 --warmup 3 --sub-timeout 5 > gpurun_out/${TAG}_n2_to.json 2> gpurun_out/${TAG}_n2_to.err
echo "n2 timeout rc=$?"; grep '^{' gpurun_out/${TAG}_n2_to.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('summa_3d'))"

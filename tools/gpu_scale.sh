#!/bin/bash
# bench.py at N = 2 and 4 (default 1D split) plus the reference arm under torchrun.
mkdir -p gpurun_out
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29800 + n)) bench.py --gpus $n > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err \
    || tail -20 gpurun_out/scale_$n.err
  grep '^{' gpurun_out/scale_$n.json | tail -1 | cut -c1-400
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29850 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/scale_ref4.json 2> gpurun_out/scale_ref4.err; echo "ref rc=$?"
grep '^{' gpurun_out/scale_ref4.json | cut -c1-300

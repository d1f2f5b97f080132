#!/bin/bash
# Redistribution throughput at p = 1, 2, 4 (run under gpurun --gpus 4).
mkdir -p gpurun_out
for n in 1 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) tools/bench_redist.py --scale ${SCALE:-20} >> gpurun_out/redist.jsonl 2> gpurun_out/redist_$n.err || tail -20 gpurun_out/redist_$n.err
done
cat gpurun_out/redist.jsonl

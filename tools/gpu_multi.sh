#!/bin/bash
# Multi-GPU evidence on an N-GPU box: the NCCL SUMMA / 3D / redistribution
# parity tests, then bench.py under torchrun for both --dist modes.
# usage: tools/gpu_multi.sh TAG N
TAG=${1:-multi}; N=${2:-4}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_redist.py -v -rs 2>&1 | tail -30 > gpurun_out/${TAG}_pytest.log
for n in $(seq 2 $N); do
  [ $n -eq 3 ] && continue
  for mode in summa 1d; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --gpus $n --dist $mode --steps 3 --warmup 3 ${BENCH_EXTRA} \
      > gpurun_out/${TAG}_bench_${mode}_$n.json 2> gpurun_out/${TAG}_bench_${mode}_$n.err
    echo "n=$n mode=$mode rc=$?"; grep '^{' gpurun_out/${TAG}_bench_${mode}_$n.json | tail -1 | cut -c1-300
  done
done
tail -5 gpurun_out/${TAG}_pytest.log

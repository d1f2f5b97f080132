#!/bin/bash
# 4-GPU evidence: NCCL drivers + C++ distributed drop-ins + distributed MCL, then bench N=2,4 (1D headline + SUMMA/3D sub-object)
TAG=${1:-r02_multi}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_redist.py tests/test_gpu_shim.py -v -rs 2>&1 | tail -25 > gpurun_out/${TAG}_pytest.log
tail -4 gpurun_out/${TAG}_pytest.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) bench.py --gpus $n --steps 5 --warmup 3 \
    > gpurun_out/${TAG}_bench_$n.json 2> gpurun_out/${TAG}_bench_$n.err
  echo "n=$n rc=$?"; grep '^{' gpurun_out/${TAG}_bench_$n.json | tail -1 | cut -c1-300
done

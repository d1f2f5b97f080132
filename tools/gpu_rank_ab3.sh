#!/bin/bash
TAG=${1:-rk5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py -x -q -k "value or tmajor or interleave or ragged or rewrite or variants" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
for cap in 8192 10240 9216 8192 10240; do
bash tools/gpu_mp.sh ${TAG}_c$cap --opt DIRECT_VALUE_RANK=$cap
done

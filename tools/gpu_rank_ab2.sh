#!/bin/bash
TAG=${1:-rk4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_value_form.py tests/test_gpu_local.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
bash tools/gpu_mp.sh ${TAG}_def
bash tools/gpu_mp.sh ${TAG}_c10k --opt DIRECT_VALUE_RANK=10240
bash tools/gpu_mp.sh ${TAG}_c12k --opt DIRECT_VALUE_RANK=12288

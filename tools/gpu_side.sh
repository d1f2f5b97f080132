#!/bin/bash
TAG=${1:-sd1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_value_form.py tests/test_gpu_local.py tests/test_gpu_mcl.py tests/test_gpu_batched.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
bash tools/gpu_mp.sh ${TAG}
bash tools/gpu_mp.sh ${TAG}b
timeout 600 python tools/bench_configs.py --configs C4 --steps 3 --warmup 2 | cut -c1-200

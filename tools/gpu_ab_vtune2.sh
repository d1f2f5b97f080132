#!/bin/bash
TAG=${1:-vt2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_value_form.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_u128.so
timeout 900 python -m pytest tests/test_gpu_direct.py -x -q -k "value or tmajor or interleave" > gpurun_out/${TAG}_pytest_u128.log 2>&1
echo "pytest u128 rc=$?"; tail -1 gpurun_out/${TAG}_pytest_u128.log
for v in prod u128 prod u128; do
  if [ $v = prod ]; then unset SLAPCU_LIB; else export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$v.so; fi
  bash tools/gpu_mp.sh ${TAG}_$v | tail -1 | sed "s/^/$v /"
done
unset SLAPCU_LIB
timeout 600 python tools/bench_configs.py --configs C4,C1 --steps 5 --warmup 3 | cut -c1-160

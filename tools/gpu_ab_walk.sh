#!/bin/bash
TAG=${1:-aw1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_value_form.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for v in prod prev prod prev; do
  if [ $v = prod ]; then unset SLAPCU_LIB; else export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$v.so; fi
  bash tools/gpu_mp.sh ${TAG}_$v | tail -1 | sed "s/^/$v /"
done

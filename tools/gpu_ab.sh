#!/bin/bash
# A/B of bench options on one box: tools/gpu_ab.sh TAG "pytest files|-" "args A" "args B" ...
TAG=$1; TESTS=$2; shift 2
mkdir -p gpurun_out
if [ "$TESTS" != "-" ]; then timeout 1200 python -m pytest $TESTS -x -q 2>&1 | tail -8 > gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_pytest.log; fi
i=0
for a in "$@"; do
  timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu --second 0 $a > gpurun_out/${TAG}_$i.json 2> gpurun_out/${TAG}_$i.err
  echo "[$i] $a rc=$?"; grep '^{' gpurun_out/${TAG}_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['class_ms_per_step'])"
  i=$((i+1))
done

#!/bin/bash
TAG=${1:-ae1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py -x -q -k "bool or window or empty" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for v in prod nopf prod nopf; do
  if [ $v = prod ]; then unset SLAPCU_LIB; else export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$v.so; fi
  timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 > gpurun_out/${TAG}_or_$v.json 2> gpurun_out/${TAG}_or_$v.err
  python - gpurun_out/${TAG}_or_$v.json $v <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
c=d['roofline'].get('class_ms_per_step',{}); print(sys.argv[2], 'OrAnd ms/step', d['ms_per_step'], 'form', c['sym_heavy'], 'emit', c['num_heavy'])
PY
done

#!/bin/bash
TAG=${1:-pk1}
mkdir -p gpurun_out
export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_pack.so
timeout 900 python -m pytest tests/test_gpu_direct.py -x -q -k "bool or variants or window" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest(pack) rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for cfg in "prod 8" "pack 8" "pack 16" "pack 32" "prod 8" "pack 16"; do
  set -- $cfg
  if [ $1 = prod ]; then unset SLAPCU_LIB; else export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$1.so; fi
  timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 --short-run $2 > gpurun_out/${TAG}_or_$1_$2.json 2> gpurun_out/${TAG}_or_$1_$2.err
  python - gpurun_out/${TAG}_or_$1_$2.json "$1 sr=$2" <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
c=d['roofline'].get('class_ms_per_step',{}); print(sys.argv[2], 'OrAnd ms/step', d['ms_per_step'], 'form', c['sym_heavy'], 'emit', c['num_heavy'])
PY
done

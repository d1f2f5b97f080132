#!/bin/bash
# Value walks: per-thread short-run threshold A/B on MinPlus C3, value pass (form 0) and value form (14).
TAG=${1:-tiny1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_value_form.py -x -q > gpurun_out/${TAG}_pytest_vf.log 2>&1
echo "pytest vf rc=$?"; tail -2 gpurun_out/${TAG}_pytest_vf.log
for cfg in "0 2" "0 8" "0 16" "0 31" "14 2" "14 16" "14 31"; do
  set -- $cfg
  timeout 600 python bench.py --semiring min_plus_i32 --second 0 --steps 3 --warmup 2 --no-e2e --no-cpu \
     --opt DIRECT_VALUE_FORM=$1 --opt DIRECT_VALUE_TINY_RUN=$2 > gpurun_out/${TAG}_vf$1_tiny$2.json 2> gpurun_out/${TAG}_vf$1_tiny$2.err
  echo "bench vf=$1 tiny=$2 rc=$?"
  python - gpurun_out/${TAG}_vf$1_tiny$2.json <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    r=d['roofline']; c=r.get('class_ms_per_step',{}); print(' ms/step', d['ms_per_step'], 'form', c.get('sym_heavy'), 'num_heavy', c.get('num_heavy'), 'bin', c.get('bin'))
except Exception as e: print('no line', e)
PY
done

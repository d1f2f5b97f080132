#!/bin/bash
TAG=${1:-bud1}
mkdir -p gpurun_out
for b in 0 90 120 0 90 120; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 --budget-gb $b > gpurun_out/${TAG}_or_$b.json 2> gpurun_out/${TAG}_or_$b.err
  python - gpurun_out/${TAG}_or_$b.json "or budget=$b" <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    c=d['roofline'].get('class_ms_per_step',{}); print(sys.argv[2], 'ms/step', d['ms_per_step'], 'batches', d['config']['column_batches'], c)
except Exception as e: print(sys.argv[2], 'fail', e)
PY
done
for b in 0 100; do
  bash tools/gpu_mp.sh ${TAG}_mp$b --budget-gb $b
done

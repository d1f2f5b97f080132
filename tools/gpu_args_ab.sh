#!/bin/bash
# A/B of bench.py runtime options: each argument is one option string ("" = defaults).
mkdir -p gpurun_out
i=0
for a in "$@"; do
  i=$((i+1))
  timeout 600 python bench.py --no-e2e --no-cpu $a > gpurun_out/argab_$i.json 2>&1
  grep "^{" gpurun_out/argab_$i.json | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$a]', d['value'], d['ms_per_step'], {k: v for k, v in d['roofline']['class_ms_per_step'].items() if v > 1})"
done

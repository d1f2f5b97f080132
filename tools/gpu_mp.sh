#!/bin/bash
# MinPlus C3 bench (short) + optional extra args
TAG=${1:-mp}; shift
mkdir -p gpurun_out
timeout 600 python bench.py --semiring min_plus_i32 --second 0 --steps 3 --warmup 2 --no-e2e --no-cpu "$@" > gpurun_out/${TAG}_mp.json 2> gpurun_out/${TAG}_mp.err
echo "bench rc=$?"
python - gpurun_out/${TAG}_mp.json <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
c=d['roofline'].get('class_ms_per_step',{}); print(' ms/step', d['ms_per_step'], 'form', c.get('sym_heavy'), 'num_heavy', c.get('num_heavy'), 'parity', d.get('parity',{}).get('all_exact'))
PY

#!/bin/bash
# Value pass changes: parity tests, then MinPlus C3 bench + ncu source view of one rank launch (s18).
TAG=${1:-rk2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_value_form.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --semiring min_plus_i32 --second 0 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/${TAG}_mp.json 2> gpurun_out/${TAG}_mp.err
echo "bench rc=$?"
python - gpurun_out/${TAG}_mp.json <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
c=d['roofline'].get('class_ms_per_step',{}); print(' ms/step', d['ms_per_step'], 'form', c.get('sym_heavy'), 'num_heavy', c.get('num_heavy'), 'parity', d.get('parity',{}).get('all_exact'))
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_item_values_rank" -c 1 \
  -o gpurun_out/${TAG}_rank python bench.py --scale 18 --semiring min_plus_i32 --second 0 --steps 1 --warmup 0 --no-e2e --no-cpu \
  > gpurun_out/${TAG}_rank.log 2>&1
echo "ncu rank rc=$?"

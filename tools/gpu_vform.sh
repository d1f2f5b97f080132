#!/bin/bash
# Value form: parity tests, then MinPlus C3 A/B (value pass vs value form at 2^13 / 2^14 rows, 256 / 512 threads).
TAG=${1:-vf1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_value_form.py -x -q > gpurun_out/${TAG}_pytest_vf.log 2>&1
echo "pytest vf rc=$?"; tail -3 gpurun_out/${TAG}_pytest_vf.log
timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_local.py tests/test_gpu_batched.py -x -q > gpurun_out/${TAG}_pytest_dir.log 2>&1
echo "pytest direct rc=$?"; tail -3 gpurun_out/${TAG}_pytest_dir.log
for cfg in "0 512" "14 512" "14 256" "13 512" "13 256"; do
  set -- $cfg
  timeout 600 python bench.py --semiring min_plus_i32 --second 0 --steps 3 --warmup 2 --no-e2e --no-cpu \
     --opt DIRECT_VALUE_FORM=$1 --value-threads $2 > gpurun_out/${TAG}_mp_vf$1_t$2.json 2> gpurun_out/${TAG}_mp_vf$1_t$2.err
  echo "bench vf=$1 t=$2 rc=$?"
  python - gpurun_out/${TAG}_mp_vf$1_t$2.json <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    r=d['roofline']; print(' ms/step', d['ms_per_step'], 'GFLOPS', d['value'], 'classes', r.get('class_ms_per_step'), 'parity', d.get('parity',{}).get('all_exact'))
except Exception as e: print('no line', e)
PY
done

#!/bin/bash
TAG=${1:-rw1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py tests/test_gpu_value_form.py tests/test_gpu_local.py tests/test_gpu_batched.py tests/test_gpu_mcl.py tests/test_gpu_scale.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for r in 1 0 1 0; do
  bash tools/gpu_mp.sh ${TAG}_r$r --opt DIRECT_VALUE_ROWS=$r | tail -1 | sed "s/^/rows=$r /"
done
timeout 600 python tools/bench_configs.py --configs C4 --steps 5 --warmup 3 --opt DIRECT_VALUE_ROWS=1 | cut -c1-200
timeout 600 python tools/bench_configs.py --configs C4 --steps 5 --warmup 3 --opt DIRECT_VALUE_ROWS=0 | cut -c1-200
timeout 900 python bench.py --semiring min_plus_i32 --second 0 --steps 2 --warmup 1 --no-e2e > gpurun_out/${TAG}_mp_parity.json 2>&1
python - gpurun_out/${TAG}_mp_parity.json <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1]); print('mp parity', d['parity'].get('all_exact'), d['ms_per_step'])
PY

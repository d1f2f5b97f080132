#!/bin/bash
TAG=${1:-tr1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shim.py tests/test_gpu_batched.py tests/test_gpu_hazards.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python - gpurun_out/${TAG}_bench.json <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
m=d['min_plus_i32']
print('or', d['ms_per_step'], d['config']['column_batches'], 'mp', m['ms_per_step'], m['config']['column_batches'], 'parity', d['parity']['all_exact'], m['parity']['all_exact'], 'e2e', d['e2e']['value'], m['e2e']['value'])
PY

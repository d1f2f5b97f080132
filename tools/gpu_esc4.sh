#!/bin/bash
TAG=${1:-esc4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_esc.py tests/test_gpu_local.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for i in 1 2; do
timeout 900 python tools/bench_configs.py --configs C2,C5,C1 --steps 5 --warmup 3 > gpurun_out/${TAG}_$i.jsonl 2>&1
python - gpurun_out/${TAG}_$i.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['ms_per_product'], 'ms', 'frac', d['step_frac_hbm'], d['parity_slice'])
PY
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv \
  python tools/bench_configs.py --configs C2 --steps 1 --warmup 1 > gpurun_out/${TAG}_c2l.log 2>&1
echo "launches rc=$?"

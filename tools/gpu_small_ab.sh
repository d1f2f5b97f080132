#!/bin/bash
TAG=${1:-sm1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_esc.py tests/test_gpu_local.py tests/test_gpu_direct.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python tools/bench_configs.py --configs C1,C2,C4,C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_cfg.jsonl 2>&1
echo "cfg rc=$?"
python - gpurun_out/${TAG}_cfg.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['ms_per_product'], 'ms', d['gflops'], 'GFLOPS frac', d['step_frac_hbm'], d['parity_slice'])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c25_launches.csv \
  python tools/bench_configs.py --configs C2,C5 --steps 1 --warmup 1 > gpurun_out/${TAG}_c25l.log 2>&1
echo "launches rc=$?"

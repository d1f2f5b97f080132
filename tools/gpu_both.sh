#!/bin/bash
# default bench lines, both semirings (short), + C2
TAG=${1:-b1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_direct.py -x -q -k "bool" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 > gpurun_out/${TAG}_or.json 2> gpurun_out/${TAG}_or.err
echo "or rc=$?"
bash tools/gpu_mp.sh ${TAG}
python - gpurun_out/${TAG}_or.json <<'PY'
import json,sys
d=json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
c=d['roofline'].get('class_ms_per_step',{}); print(' OrAnd ms/step', d['ms_per_step'], c)
PY
timeout 600 python tools/bench_configs.py --configs C2 --steps 5 --warmup 3 | cut -c1-200

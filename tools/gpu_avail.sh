#!/bin/bash
TAG=${1:-av1}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_esc.py tests/test_gpu_local.py tests/test_gpu_batched.py tests/test_gpu_shim.py tests/test_gpu_gen_merge.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
for i in 1 2 3; do
timeout 900 python tools/bench_configs.py --configs C1,C2,C4,C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_$i.jsonl 2>&1
python - gpurun_out/${TAG}_$i.jsonl <<'PY'
import json,sys
print(' | '.join(f"{d['config']} {d['ms_per_product']}" for d in (json.loads(l) for l in open(sys.argv[1]) if l.startswith('{'))))
PY
done

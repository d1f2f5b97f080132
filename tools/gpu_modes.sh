mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_direct.py -x -q 2>&1 | tail -3
for m in 0 1 2; do
timeout 300 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 --mark-mode $m "$@" > gpurun_out/mode$m.log 2>&1
python - <<PY
import json; d=json.loads(open("gpurun_out/mode$m.log").read().strip().splitlines()[-1])
print("mode $m", d["ms_per_step"], d["roofline"]["class_ms_per_step"])
PY
done

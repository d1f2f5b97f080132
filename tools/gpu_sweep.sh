# Runs the bench once per argument set (separated by ';'), prints ms/step and
# the per-class device time.  Usage: bash tools/gpu_sweep.sh "--a 1;--a 2"
mkdir -p gpurun_out
[ -n "$TESTS" ] && timeout 300 python -m pytest $TESTS -x -q 2>&1 | tail -2
IFS=';' read -ra SETS <<< "$1"
i=0
for a in "${SETS[@]}"; do
  timeout 300 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 $a > gpurun_out/sweep$i.log 2>&1
  python - "$a" gpurun_out/sweep$i.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"[{sys.argv[1]}] {d['ms_per_step']} ms {d['value']} GF", {k: v for k, v in d['roofline']['class_ms_per_step'].items() if v > 0.5})
except Exception as e:
    print(f"[{sys.argv[1]}] failed: {open(sys.argv[2]).read()[-800:]}")
PY
  i=$((i+1))
done

# Runs the bench once per argument set (separated by ';'), prints ms/step and
# the per-class device time.  Usage: bash tools/gpu_sweep.sh "--a 1;--a 2"
mkdir -p gpurun_out
[ -n "$TESTS" ] && timeout 300 python -m pytest $TESTS -x -q 2>&1 | tail -2
IFS=';' read -ra SETS <<< "$1"
i=0
for a in "${SETS[@]}"; do
  timeout ${RUN_TIMEOUT:-240} python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 $a > gpurun_out/sweep$i.log 2>&1
  python tools/sweep_line.py "$a" gpurun_out/sweep$i.log
  i=$((i+1))
done

# one full ncu capture of a named kernel in the bench command.
# Usage: bash tools/gpu_prof1.sh TAG KERNEL_REGEX SKIP [bench args]
set -x
mkdir -p gpurun_out
TAG=$1; KRE=$2; SKIP=$3; shift 3
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 1 \
  -o gpurun_out/${TAG} python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/${TAG}_run.log 2>&1
ls -la gpurun_out

# ncu evidence for the bench command: launch list (durations only) and one
# full capture of the top kernels.  Usage: bash tools/gpu_prof.sh TAG [bench args]
set -x
mkdir -p gpurun_out
TAG=${1:-prof}; shift
ARGS="$@"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu $ARGS > gpurun_out/${TAG}_launch_run.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_fused|k_copy' -s 20 -c 4 \
  -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e $ARGS > gpurun_out/${TAG}_full_run.log 2>&1
ls -la gpurun_out

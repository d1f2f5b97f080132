# Round evidence for the default bench command: launch list + one full ncu
# capture of each of the two top kernels.  Usage: bash tools/gpu_prof3.sh TAG [bench args]
set -x
mkdir -p gpurun_out
TAG=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/${TAG}_launch_run.log 2>&1
for k in k_tile_form k_tile_emit; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
  -o gpurun_out/${TAG}_${k} python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/${TAG}_${k}_run.log 2>&1
done
ls -la gpurun_out | tail -5

set -x
mkdir -p gpurun_out
TAG=$1; shift
[ -n "$NOLAUNCH" ] || timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/${TAG}_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_tile_form}" -s 4 -c 1 \
  -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/${TAG}_full_run.log 2>&1
ls -la gpurun_out

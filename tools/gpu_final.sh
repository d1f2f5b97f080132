#!/bin/bash
# Final-build evidence on one GPU: the driver's bench command, an ncu launch list of the
# same workload, and ncu --set full captures of the form+emit pair (same batch) for
# OrAnd and of form+emit+values for MinPlus int32.
TAG=${1:-r02_final}
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 > gpurun_out/${TAG}_launch_run.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_mp_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 --semiring min_plus_i32 > gpurun_out/${TAG}_mp_launch_run.log 2>&1
echo "mp launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tile_form|k_tile_emit" -s 10 -c 2 \
  -o gpurun_out/${TAG}_pair python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 > gpurun_out/${TAG}_pair.log 2>&1
echo "pair rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_tile_form|k_tile_emit|k_item_values_rank" -s 15 -c 3 \
  -o gpurun_out/${TAG}_mp python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 --semiring min_plus_i32 > gpurun_out/${TAG}_mp.log 2>&1
echo "mp rc=$?"
grep '^{' gpurun_out/${TAG}_bench.json | cut -c1-400

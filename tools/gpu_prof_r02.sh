#!/bin/bash
# ncu --set full captures of the hot kernels (one launch each), with source.
mkdir -p gpurun_out
T=${TAG:-r02_prof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_form -s 5 -c 1 \
  -o gpurun_out/${T}_form python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 $BARGS > gpurun_out/${T}_form.log 2>&1
echo "form rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_item_values_rank -s 9 -c 1 \
  -o gpurun_out/${T}_vrank python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 --semiring min_plus_i32 $BARGS > gpurun_out/${T}_vrank.log 2>&1
echo "vrank rc=$?"
ls -la gpurun_out | grep $T

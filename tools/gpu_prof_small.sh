#!/bin/bash
# ncu source captures: ESC expand (C5), light hash (C2), emit (OrAnd s18)
TAG=${1:-ps1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_expand" -c 1 \
  -o gpurun_out/${TAG}_c5exp python tools/bench_configs.py --configs C5 --steps 1 --warmup 0 > gpurun_out/${TAG}_c5.log 2>&1
echo "c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused_light" -c 2 \
  -o gpurun_out/${TAG}_c2light python tools/bench_configs.py --configs C2 --steps 1 --warmup 0 > gpurun_out/${TAG}_c2.log 2>&1
echo "c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile_emit|k_tile_form" -c 2 \
  -o gpurun_out/${TAG}_pair python bench.py --scale 18 --steps 1 --warmup 0 --no-e2e --no-cpu --second 0 > gpurun_out/${TAG}_pair.log 2>&1
echo "pair rc=$?"

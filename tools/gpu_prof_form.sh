#!/bin/bash
# one ncu --set full capture of k_tile_form with bench args $BARGS, tag $TAG; then an A/B list
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-k_tile_form} -s ${SKIP:-5} -c 1 \
  -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 $BARGS > gpurun_out/${TAG}_full.log 2>&1
echo "ncu rc=$?"

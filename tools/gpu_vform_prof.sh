#!/bin/bash
# ncu of one k_value_form launch (MinPlus, R-MAT s18) at 2^14 / 512 threads, and launch lists of C2 / C5.
TAG=${1:-vfp1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_value_form" -c 1 \
  -o gpurun_out/${TAG}_vform python bench.py --scale 18 --semiring min_plus_i32 --second 0 --steps 1 --warmup 0 --no-e2e --no-cpu \
  > gpurun_out/${TAG}_vform.log 2>&1
echo "ncu vform rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv \
  python tools/bench_configs.py --configs C2 --steps 1 --warmup 1 > gpurun_out/${TAG}_c2.log 2>&1
echo "c2 launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c5_launches.csv \
  python tools/bench_configs.py --configs C5 --steps 1 --warmup 1 > gpurun_out/${TAG}_c5.log 2>&1
echo "c5 launches rc=$?"
timeout 600 python tools/bench_configs.py --configs C2,C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_c25.jsonl 2>&1
echo "c2c5 rc=$?"; cut -c1-300 gpurun_out/${TAG}_c25.jsonl

#!/bin/bash
# Final evidence of the late round-2 build on one GPU: full GPU tests, smoke, the driver's bench
# command (both arms), launch lists, ncu --set full of the same batches (traffic), secondary configs.
TAG=${1:-r02_final6}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 > gpurun_out/${TAG}_launch_run.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_mp_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 --semiring min_plus_i32 > gpurun_out/${TAG}_mp_launch_run.log 2>&1
echo "mp launches rc=$?"
# skip exactly one warm-up step's launches, so the captured kernels are batch 0 of the second step
NB=$(python -c "import json;print([json.loads(l) for l in open('gpurun_out/${TAG}_bench.json') if l.startswith('{')][-1]['config']['column_batches'])")
NBM=$(python -c "import json;print([json.loads(l) for l in open('gpurun_out/${TAG}_bench.json') if l.startswith('{')][-1]['min_plus_i32']['config']['column_batches'])")
echo "batches $NB minplus $NBM"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tile_form|k_tile_emit" -s $((2 * NB)) -c 2 \
  -o gpurun_out/${TAG}_pair python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 > gpurun_out/${TAG}_pair.log 2>&1
echo "pair rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_tile_form|k_tile_emit|k_item_values_rank" -s $((3 * NBM)) -c 3 \
  -o gpurun_out/${TAG}_mp python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --second 0 --semiring min_plus_i32 > gpurun_out/${TAG}_mp.log 2>&1
echo "mp rc=$?"
timeout 900 python tools/bench_configs.py --configs C1,C2,C4,C5 --steps 5 --warmup 3 > gpurun_out/${TAG}_configs.jsonl 2>&1
echo "configs rc=$?"
grep '^{' gpurun_out/${TAG}_bench.json | cut -c1-400

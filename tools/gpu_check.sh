#!/bin/bash
# quick GPU check: selected pytest files, then bench at a small and the full scale
# usage: tools/gpu_check.sh TAG "pytest files" "bench args"
TAG=${1:-chk}; TESTS=${2:-tests/test_gpu_hazards.py}; BARGS=${3:-}
mkdir -p gpurun_out
free -g | head -2 > gpurun_out/${TAG}_host.txt; nproc >> gpurun_out/${TAG}_host.txt
timeout 900 python -m pytest $TESTS -x -q 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --scale 16 --steps 3 --warmup 3 $BARGS > gpurun_out/${TAG}_bench16.json 2> gpurun_out/${TAG}_bench16.err
echo "bench16 rc=$?"
timeout 1200 python bench.py --steps 10 --warmup 3 $BARGS > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log; tail -3 gpurun_out/${TAG}_bench16.err gpurun_out/${TAG}_bench.err

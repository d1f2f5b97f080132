set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_direct.py -x -q > gpurun_out/direct_tests.log 2>&1
tail -30 gpurun_out/direct_tests.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/direct_bench.log 2>&1
tail -5 gpurun_out/direct_bench.log

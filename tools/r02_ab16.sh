timeout 900 python -m pytest tests/test_gpu_direct.py tests/test_gpu_hazards.py -k "value" -x -q 2>&1 | tail -1
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab16_$1.json 2>&1; grep '^{' gpurun_out/r02_ab16_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
run mp "--semiring min_plus_i32"
timeout 600 python tools/bench_configs.py --configs C4 2>/dev/null | cut -c1-200

timeout 900 python -m pytest tests/test_gpu_direct.py -k "value" -x -q 2>&1 | tail -2
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab10_$1.json 2>&1; grep '^{' gpurun_out/r02_ab10_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
run mp "--semiring min_plus_i32"
run mp_do "--semiring min_plus_i32 --opt DIRECT_VALUE_DENSE_ONLY=1"
run mp_do4 "--semiring min_plus_i32 --opt DIRECT_VALUE_DENSE_ONLY=1 --value-rank 4096"
run mp_sub13 "--semiring min_plus_i32 --value-rank 0 --value-tile-log2 13"

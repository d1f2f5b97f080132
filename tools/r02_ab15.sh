run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab15_$1.json 2>&1; grep '^{' gpurun_out/r02_ab15_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
run base ""
run mp512 "--semiring min_plus_i32"
run mp256 "--semiring min_plus_i32 --value-threads 256"
run mp256c4 "--semiring min_plus_i32 --value-threads 256 --value-rank 4096"

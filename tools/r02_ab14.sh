run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab14_$1.json 2>&1; grep '^{' gpurun_out/r02_ab14_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
timeout 900 python -m pytest tests/test_gpu_direct.py -x -q 2>&1 | tail -1
run ipw128 ""
SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_ipw64.so run ipw64 ""
SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_ipw256.so run ipw256 ""
run mp "--semiring min_plus_i32"

run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab13_$1.json 2>&1; grep '^{' gpurun_out/r02_ab13_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
timeout 600 python -m pytest tests/test_gpu_direct.py -x -q -k "bool" 2>&1 | tail -1
run nt64 ""
SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_emitnt32.so run nt32 ""
run nt64b ""

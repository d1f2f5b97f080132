timeout 900 python -m pytest tests/test_gpu_esc.py -x -q 2>&1 | tail -2
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab9_$1.json 2>&1; grep '^{' gpurun_out/r02_ab9_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
run mp "--semiring min_plus_i32"
SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_vtiny0.so run mp_t0 "--semiring min_plus_i32"
SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_vtiny4.so run mp_t4 "--semiring min_plus_i32"
timeout 900 python tools/bench_configs.py > gpurun_out/r02_ab9_cfg.jsonl 2>gpurun_out/r02_ab9_cfg.err
python -c "
import json
for l in open('gpurun_out/r02_ab9_cfg.jsonl'):
    d=json.loads(l); print(d['config'], d['ms_per_product'], d['gflops'], d['step_frac_hbm'], d['parity_slice'])"

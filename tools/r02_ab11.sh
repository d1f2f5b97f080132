timeout 900 python -m pytest tests/test_gpu_direct.py -k "value_l2 or value_pass" -x -q 2>&1 | tail -2
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab11_$1.json 2>&1; grep '^{' gpurun_out/r02_ab11_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
run base ""
run mp "--semiring min_plus_i32"
run mp_l2 "--semiring min_plus_i32 --opt DIRECT_VALUE_L2=1"
timeout 900 python tools/bench_configs.py --configs C1,C4 --opt DIRECT_VALUE_L2=1 > gpurun_out/r02_ab11_cfg_l2.jsonl 2>&1
timeout 900 python tools/bench_configs.py --configs C1,C4 > gpurun_out/r02_ab11_cfg.jsonl 2>&1
for f in gpurun_out/r02_ab11_cfg.jsonl gpurun_out/r02_ab11_cfg_l2.jsonl; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'): d=json.loads(l); print('$f'[-12:], d['config'], d['ms_per_product'], d['parity_slice'])"; done

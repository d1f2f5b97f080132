timeout 900 python -m pytest tests/test_gpu_esc.py -x -q 2>&1 | tail -3
timeout 900 python tools/bench_configs.py --opt DIRECT_ESC=1 --configs C1,C2,C5 > gpurun_out/r02_c10_cfg_esc.jsonl 2>gpurun_out/r02_c10_cfg_esc.err
cut -c1-200 gpurun_out/r02_c10_cfg_esc.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c10_c2esc_launches.csv python tools/bench_configs.py --configs C2 --steps 1 --warmup 0 --opt DETERMINISTIC=1 > /dev/null 2>&1
SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_vcount.so timeout 600 python tools/vcount.py 20
for v in "" emit10 emit9; do
  if [ -n "$v" ]; then export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$v.so; else unset SLAPCU_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 > gpurun_out/r02_c10_emit_$v.json 2>&1
  grep '^{' gpurun_out/r02_c10_emit_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['class_ms_per_step'])"
done

run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --second 0 $2 > gpurun_out/r02_ab12_$1.json 2>&1; grep '^{' gpurun_out/r02_ab12_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['roofline']['class_ms_per_step'])"; }
run base ""
for v in emitnt64 emitnt256 formu8 unit512 unit128; do SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$v.so run $v ""; done
run base2 ""

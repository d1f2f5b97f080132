#!/bin/bash
# A/B of variant libraries on the default bench (no e2e / cpu legs).
# Usage: bash tools/gpu_ab.sh name1 name2 ...   ("base" = the product library)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then L=""; else L=paper_2106_14402_b200/variants/libslapcu_$v.so; fi
  SLAPCU_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/ab_$v.json 2>&1
  grep "^{" gpurun_out/ab_$v.json | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], {k: v for k, v in d['roofline']['class_ms_per_step'].items() if v > 1})"
done

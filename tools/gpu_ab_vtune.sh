#!/bin/bash
TAG=${1:-vt1}
mkdir -p gpurun_out
for cfg in "prod 2" "prod 0" "prod 1" "prod 4" "u512 2" "u128 2" "prod 2"; do
  set -- $cfg
  if [ $1 = prod ]; then unset SLAPCU_LIB; else export SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_$1.so; fi
  bash tools/gpu_mp.sh ${TAG}_$1_$2 --opt DIRECT_VALUE_TINY_RUN=$2 | tail -1 | sed "s/^/$1 tiny=$2 /"
done

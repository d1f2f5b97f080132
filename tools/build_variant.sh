#!/bin/bash
# A/B build: recompile direct.cu with extra -D flags and link a variant library
# next to the product one.  Usage: bash tools/build_variant.sh NAME -DFOO=1 ...
# then run with SLAPCU_LIB=paper_2106_14402_b200/variants/libslapcu_NAME.so
set -e
NAME=$1; shift
python -c "from paper_2106_14402_b200 import _build; _build.build(verbose=False)"
mkdir -p paper_2106_14402_b200/variants build/variant
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr --extended-lambda -Xcompiler -fPIC,-O3 -Iinclude -Ipaper_2106_14402_b200/csrc"
nvcc $FLAGS "$@" -c paper_2106_14402_b200/csrc/direct.cu -o build/variant/direct_$NAME.o
OBJS=$(ls build/obj/*.o | grep -v '/direct.cu.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2106_14402_b200/variants/libslapcu_$NAME.so $OBJS build/variant/direct_$NAME.o -lnccl -lcudart
ls -la paper_2106_14402_b200/variants/libslapcu_$NAME.so

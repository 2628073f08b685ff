#!/bin/bash
# Dev helper: experiment builds of libqapsa with -DTC_EXP=<bits> into tools/libqapsa_exp<bits>.so
cd "$(dirname "$0")/.."
for b in "$@"; do
  nvcc -DTC_EXP=$b -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
    -Xcompiler -fPIC -Xcompiler -ffp-contract=off -shared -cudart static -I include \
    -o tools/libqapsa_exp$b.so paper_1208_2675_b200/csrc/qapsa.cu || exit 1
done

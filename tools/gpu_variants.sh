#!/bin/bash
# time config 3 (1e8) on the in-tree library and on every variants/libqapsa_*.so (dev helper)
mkdir -p gpurun_out
OUT=gpurun_out/variants.log
: > $OUT
for lib in paper_1208_2675_b200/libqapsa.so variants/libqapsa_*.so; do
  for i in 1 2; do
    echo -n "$(basename $lib) " >> $OUT
    QAPSA_LIB=$PWD/$lib timeout 100 python tools/run_cfg3.py ${ITERS:-1e8} >> $OUT 2>&1
  done
done

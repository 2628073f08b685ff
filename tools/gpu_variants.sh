#!/bin/bash
# time a command (default: config 3, 1e8) on the in-tree library and on every
# variants/libqapsa_*.so (dev helper): CMD="python tools/run_ens.py 8192 1e7" bash tools/gpu_variants.sh
mkdir -p gpurun_out
OUT=gpurun_out/variants.log
CMD=${CMD:-python tools/run_cfg3.py 1e8}
: > $OUT
for lib in paper_1208_2675_b200/libqapsa.so variants/libqapsa_*.so; do
  for i in 1 2; do
    echo -n "$(basename $lib) " >> $OUT
    QAPSA_LIB=$PWD/$lib timeout 100 $CMD >> $OUT 2>&1
  done
done

#!/bin/bash
OUT=gpurun_out
for g in 16384 65536 262144 1048576 2147483647; do
  timeout 300 python tools/run_ens.py 8192 1e7 0 $g 1 >> $OUT/ens_gap.log 2>&1
done
echo done

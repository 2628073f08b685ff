#!/bin/bash
# ncu --set full (with source) of the scratch phase on config 3's hot start
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 120 python tools/run_cfg3.py 2e5 > $OUT/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sa_scratch -c 1 \
    -o $OUT/prof_sa_scratch_${TAG:-q} python tools/run_cfg3.py 2e5 > $OUT/ncu_full.log 2>&1
echo done

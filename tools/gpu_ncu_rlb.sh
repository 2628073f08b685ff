#!/bin/bash
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 120 python tools/run_cfg.py 4 2e5 > $OUT/prof_plain_rlb.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_relabel -c 1 \
    -o $OUT/prof_relabel_${TAG:-q} python tools/run_cfg.py 4 2e5 > $OUT/ncu_full_rlb.log 2>&1
echo done

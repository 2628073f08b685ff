#!/bin/bash
# ensemble (config 5): launch list of the full run and one ncu --set full of the scratch phase
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python tools/run_ens.py 8192 1e7 > $OUT/ens_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/ens_launches.csv python tools/run_ens.py 8192 1e7 > $OUT/ens_ncu.log 2>&1
timeout 120 python tools/run_ens.py 1184 2e5 > $OUT/prof_plain_ens.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_scratch -c 1 \
    -o $OUT/prof_ens_${TAG:-q} python tools/run_ens.py 1184 2e5 > $OUT/ncu_full_ens.log 2>&1
echo done

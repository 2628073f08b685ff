#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -k "relabel or grey or uint16 or twin or engine_selection or qaplib or smoke" -x > $OUT/pytest_rlb.log 2>&1; echo "rc=$?" >> $OUT/pytest_rlb.log
timeout 300 python tools/run_cfg.py 4 1e7 > $OUT/cfg4_1e7.log 2>&1
timeout 300 python tools/run_cluster.py 512 1e6 > $OUT/cluster512.log 2>&1
echo done

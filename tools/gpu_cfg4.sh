#!/bin/bash
# relabel engine (config 4): parity tests, prefix timing, optionally the full-run goldens (FULL=1)
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -k "relabel or grey or uint16 or twin or engine_selection" -x > $OUT/pytest_rlb.log 2>&1; echo "rc=$?" >> $OUT/pytest_rlb.log
timeout 300 python tools/run_cfg.py 4 1e7 > $OUT/cfg4_1e7.log 2>&1
timeout 300 python tools/run_cfg.py 4 1e6 > $OUT/cfg4_1e6.log 2>&1
if [ "${FULL:-0}" = 1 ]; then
  timeout 1200 python -m pytest tests -q -m gpu -k "config4_full" -x --durations=3 > $OUT/pytest_cfg4_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_cfg4_full.log
fi
echo done

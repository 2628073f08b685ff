#!/bin/bash
# full GPU parity pass including the long golden tests (config 4 full 1e9, all config-5 chains)
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rA --durations=15 > $OUT/pytest_gpu_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_full.log
echo done

#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -k "cluster" -x > $OUT/pytest_cluster.log 2>&1; echo "rc=$?" >> $OUT/pytest_cluster.log
echo done

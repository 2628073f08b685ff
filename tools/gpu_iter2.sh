#!/bin/bash
# relabel / cluster iteration: their parity tests, config-4 prefix, N = 512
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "relabel or grey or cluster or near_tie or config4_prefix" > gpurun_out/it2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/it2_tests.log
timeout 300 python tools/run_cfg.py 4 1e7 > gpurun_out/it2_cfg4.log 2>&1
timeout 300 python tools/run_cluster.py 512 1e6 > gpurun_out/it2_clu.log 2>&1

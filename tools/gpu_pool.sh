#!/bin/bash
# device-pool change: e2e breakdown + new test + quick regression subset
mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py 6 bench > gpurun_out/e2e.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pool or config1 or config2 or ensemble_four or cluster_engine_n512 or switch_gap" > gpurun_out/pool_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_pool.log 2>&1

#!/bin/bash
# one optimisation iteration: parity subset, bench (config 3 + ensemble + config-4 prefix)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "not goldens and not slow" > gpurun_out/it_tests.log 2>&1; echo "rc=$?" >> gpurun_out/it_tests.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err

#!/bin/bash
# phase timers of the scratch phase over config 3's full run and its first 2e5 iterations
mkdir -p gpurun_out
python -c "from paper_1208_2675_b200 import _build; _build.build(timers=True)" > gpurun_out/timers_build.log 2>&1
timeout 120 python tools/scratch_phase.py 1e8 > gpurun_out/scratch_phase_full.log 2>&1
timeout 120 python tools/scratch_phase.py 2e5 > gpurun_out/scratch_phase.log 2>&1

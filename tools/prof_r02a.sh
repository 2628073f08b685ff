#!/bin/bash
# round-2 profiling pass: phase timers of the scratch phase, ensemble launch list, full ncu of the
# scratch phase (hot start) and the Δ engine (cold tail), with source.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_1208_2675_b200 import _build; _build.build(timers=True)" > $OUT/timers_build.log 2>&1
timeout 120 python tools/scratch_phase.py 2e5 > $OUT/scratch_phase.log 2>&1
timeout 120 python tools/phase_tc.py 2e6 3e7 > $OUT/phase_tc_cold.log 2>&1
timeout 300 python tools/run_ens.py 8192 1e7 > $OUT/ens_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/ens_launches.csv python tools/run_ens.py 8192 1e7 > $OUT/ens_ncu.log 2>&1
timeout 120 python tools/run_cfg3.py 2e5 > $OUT/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sa_scratch -c 1 \
    -o $OUT/prof_sa_scratch_r02 python tools/run_cfg3.py 2e5 > $OUT/ncu_full.log 2>&1
timeout 120 python tools/run_cfg3.py 2e6 3e7 > $OUT/prof_plain_tc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_tc -c 1 \
    -o $OUT/prof_sa_tc_r02 python tools/run_cfg3.py 2e6 3e7 > $OUT/ncu_full_tc.log 2>&1
echo done

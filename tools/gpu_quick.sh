#!/bin/bash
# quick GPU pass: parity (without the long golden tests), bench, phase timers; optional ncu of
# the scratch phase (NCU=1) and the Δ engine's tail (NCU_TC=1)
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -k "not goldens" -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
python -c "from paper_1208_2675_b200 import _build; _build.build(timers=True)" > $OUT/timers_build.log 2>&1
timeout 120 python tools/scratch_phase.py 2e5 > $OUT/scratch_phase.log 2>&1
timeout 120 python tools/phase_tc.py 2e6 3e7 > $OUT/phase_tc_cold.log 2>&1
timeout 120 python tools/run_cfg3.py 1e8 > $OUT/cfg3_plain.log 2>&1
if [ "${NCU:-0}" = 1 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sa_scratch -c 1 \
    -o $OUT/prof_sa_scratch_q python tools/run_cfg3.py 2e5 > $OUT/ncu_full.log 2>&1
fi
if [ "${NCU_TC:-0}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_tc -c 1 \
    -o $OUT/prof_sa_tc_q python tools/run_cfg3.py 2e6 3e7 > $OUT/ncu_full_tc.log 2>&1
fi
echo done

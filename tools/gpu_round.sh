#!/bin/bash
# One GPU-box session: tests, bench, ncu launch list + full captures (see B200_PROFILING.md).
# Usage (via gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# launch list of the timed single-chain workload (same command plain, then under ncu)
CMD="python bench.py --steps 2 --warmup 3 --no-ensemble --no-cpu-baseline --no-config4 --e2e-steps 1"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_launch.log
# full captures: the scratch phase (dominant) on config 3's hot start, the Δ engine on its tail
timeout 120 python tools/run_cfg3.py 2e5 > $OUT/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sa_scratch -c 1 \
    -o $OUT/prof_sa_scratch_$TAG python tools/run_cfg3.py 2e5 > $OUT/ncu_full.log 2>&1
echo "full scratch rc=$?" >> $OUT/ncu_full.log
timeout 120 python tools/run_cfg3.py 2e6 3e7 > $OUT/prof_plain_tc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_tc -c 1 \
    -o $OUT/prof_sa_tc_$TAG python tools/run_cfg3.py 2e6 3e7 > $OUT/ncu_full_tc.log 2>&1
echo "full tc rc=$?" >> $OUT/ncu_full_tc.log
# relabel engine (config 4 hot start) and the tensor-memory ensemble's scratch phase
timeout 120 python tools/run_cfg.py 4 5e4 0 > $OUT/prof_plain_rlb.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_relabel -c 1 \
    -o $OUT/prof_relabel_$TAG python tools/run_cfg.py 4 5e4 0 > $OUT/ncu_full_rlb.log 2>&1
echo "full relabel rc=$?" >> $OUT/ncu_full_rlb.log
timeout 120 python tools/run_ens.py 1184 2e5 > $OUT/prof_plain_ens.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:k_sa_scratch -c 1 \
    -o $OUT/prof_ens_$TAG python tools/run_ens.py 1184 2e5 > $OUT/ncu_full_ens.log 2>&1
echo "full ensemble rc=$?" >> $OUT/ncu_full_ens.log

#!/bin/bash
# round-end evidence: full GPU parity (incl. goldens), smoke, bench (ours + reference arm),
# kernel launch lists of the timed workloads, random-proposal timing
set -u
OUT=gpurun_out
mkdir -p $OUT/final
F=$OUT/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $F/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rA --durations=10 > $F/pytest_gpu.log 2>&1; echo "rc=$?" >> $F/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo "rc=$?" >> $F/smoke.log
timeout 900 python bench.py > $F/bench.json 2> $F/bench.err; echo "rc=$?" >> $F/bench.err
timeout 600 python bench.py --impl reference > $F/bench_ref.json 2> $F/bench_ref.err; echo "rc=$?" >> $F/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-ensemble --no-cpu-baseline --no-config4 --e2e-steps 1"
timeout 300 $CMD > $F/plain_cfg3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $F/launches_cfg3.csv $CMD > $F/ncu_cfg3.log 2>&1
timeout 300 python tools/run_ens.py 8192 1e7 > $F/plain_ens.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $F/launches_ens.csv python tools/run_ens.py 8192 1e7 > $F/ncu_ens.log 2>&1
timeout 300 python tools/run_rnd.py 1e7 > $F/rnd.log 2>&1
timeout 300 python tools/run_cluster.py 512 1e6 > $F/cluster512.log 2>&1
echo done

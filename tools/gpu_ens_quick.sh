OUT=gpurun_out
timeout 600 python bench.py --no-config4 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/ens_launches.csv python tools/run_ens.py 8192 1e7 > $OUT/ens_ncu.log 2>&1
echo done

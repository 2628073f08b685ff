#!/bin/bash
# round profiling pass: ncu --set full (with source) of every hot kernel, each after its plain run;
# summarised on the box (tools/ncu_summarize.py -> gpurun_out/prof/), the .ncu-rep files deleted
# (the 64 MiB return limit) unless KEEP=1
set -u
OUT=gpurun_out
TAG=${TAG:-r02}
mkdir -p $OUT/prof
cap() {  # name kernel-regex units command...
  local name=$1 kre=$2 units=$3; shift 3
  timeout 300 "$@" > $OUT/prof/plain_$name.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 \
      -o $OUT/prof_${name}_$TAG "$@" > $OUT/prof/ncu_$name.log 2>&1
  echo "$name rc=$?" >> $OUT/prof/profiles_rc.log
  OUTDIR=$OUT/prof python tools/ncu_summarize.py $TAG $name=$OUT/prof_${name}_$TAG.ncu-rep:$units >> $OUT/prof/summarize.log 2>&1
  [ "${KEEP:-0}" = 1 ] || rm -f $OUT/prof_${name}_$TAG.ncu-rep
}
case "${WHICH:-all}" in
  all|single) cap k_sa_scratch k_sa_scratch 37828 python tools/run_cfg3.py 2e5
              cap k_sa_tc k_sa_tc 1 python tools/run_cfg3.py 2e6 3e7 ;;
esac
case "${WHICH:-all}" in
  all|ens) cap k_ens_scratch k_ens_scratch 1 python tools/run_ens.py 1184 2e5 ;;
esac
case "${WHICH:-all}" in
  all|big) cap k_sa_relabel k_sa_relabel 1 python tools/run_cfg.py 4 2e5
           cap k_sa_cluster k_sa_cluster 1 python tools/run_cluster.py 512 2e5 ;;
esac
echo done

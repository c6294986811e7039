#!/bin/bash
# tile-height (T1) variant sweep for K1 (development).
run() { echo "N=$1 SO=$2 T1=$3 UNR=${4:-def}: $(SWB_T1=$3 ${4:+SWB_UNR=$4} timeout 60 python scripts/probe_perf.py factorised $2 $1 ${NT:-200} 2>&1 | tail -1 | sed 's/form=factorised *//')"; }
for n in 256 512; do
  run $n 4 30; run $n 4 28
  run $n 8 30; run $n 8 28
  run $n 12 30; run $n 12 28; run $n 12 28 4; run $n 12 26
  run $n 16 22; run $n 16 20
done

#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_cases.py); logs in gpurun_out/sanitize_*.log
# (summaries copied to profiles/sanitize_r02.txt).  Each tool reports "ERROR SUMMARY: 0 errors" when clean.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  cases=${CASES:-"k1 pencil simple slabs extras"}
  # initcheck serialises co-resident grids: the fused-ordering slabs would hit their 20 s bounded wait
  [ $tool = initcheck ] && cases=${CASES_INIT:-"k1 pencil_single simple slabs_ordered extras"}
  for case in $cases; do
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py $case \
        > gpurun_out/sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${case}.log | tail -1)"
  done
done

#!/bin/bash
# ncu evidence for the stencil kernels (run under gpurun; one GPU).
#  1. launch list of the bench command (per-kernel share of the step)
#  2. one --set full capture of K1 (k_tma, one step per launch) per space order
set -x
mkdir -p gpurun_out
# the driver's default bench command; ncu records the first 400 kernel launches (setup, the
# 10 warm-up steps and 380+ timed steps), the rest of the run executes unprofiled
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py > gpurun_out/launches_bench.log 2>&1
for so in ${SOS:-4 8 12 16}; do
  ncu --set full --clock-control none --import-source on -k regex:k_tma -s 6 -c 1 \
      -o gpurun_out/tma_so$so python scripts/probe_perf.py factorised $so 256 8 > gpurun_out/ncu_so$so.log 2>&1
done

#!/bin/bash
# One ncu --set full capture with source of the k_tma kernel per SO (256^3), for the source page.
mkdir -p gpurun_out
for so in ${SOS:-8 16}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tma -s 6 -c 1 \
      -o gpurun_out/${TAG:-tma}_so$so python scripts/probe_perf.py factorised $so 256 8 > gpurun_out/ncu_${TAG:-tma}_so$so.log 2>&1
  echo "so $so rc=$?"
done

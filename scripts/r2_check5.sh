#!/bin/bash
mkdir -p gpurun_out
V=paper_1912_00695_b200/_lib/variants
for lib in $V/libswb_dither.so $V/libswb_dither_lap2.so; do
  SWB_LIB=$lib timeout 600 python scripts/probe_combine.py
done 2>&1 | tee gpurun_out/dither.log
for i in 1 2; do
TAG=base timeout 300 python scripts/probe_k1perf.py 256:12 256:16 512:12 512:16
SWB_LIB=$V/libswb_lap1b.so TAG=lap1 timeout 300 python scripts/probe_k1perf.py 256:12 256:16 512:12 512:16
done 2>&1 | tee gpurun_out/lap1perf.log

#!/bin/bash
# SO 12 pencil split point with P_y through the aux ring: k >= 4 (default) vs k >= 3 / 5 (variant builds
# k6_3 / k6_5: build.py --variant k6_3 -DSWB_PENCIL_K6=3).
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for lib in "" ${VARIANTS:-k6_3 k6_5}; do
    if [ -n "$lib" ]; then export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so; else unset SWB_LIB; fi
    timeout 300 python scripts/probe_k1perf.py 256:12 384:12 512:12
  done
done

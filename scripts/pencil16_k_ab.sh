#!/bin/bash
# SO 16 pencil split point with P_y through the aux ring: k >= 4 (default) vs k >= 3 / 5 (variant builds k3 / k5:
# build.py --variant k3 -DSWB_PENCIL_K=3; the override applies to every halo, only the SO 16 lines matter).
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for lib in "" k3 k5; do
    if [ -n "$lib" ]; then export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so; else unset SWB_LIB; fi
    timeout 300 python scripts/probe_k1perf.py 256:16 512:16
  done
done

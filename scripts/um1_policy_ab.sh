#!/bin/bash
# L2 policy of the u[t-1] aux load: evict_first (default) vs normal (-DSWB_UM1_NORMAL=1 build of the A/B; the switch was folded into k_tma.cu as "normal at H >= 8").
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for lib in "" um1n; do
    if [ -n "$lib" ]; then export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so; else unset SWB_LIB; fi
    timeout 300 python scripts/probe_k1perf.py 256:8 256:12 256:16 512:8 512:16
  done
done

#!/bin/bash
# u[t+1] row-store L2 policy: evict_last 1.0 (default) vs evict_last 0.5 (el05) vs evict_normal (elnorm); the switches
# (SWB_EL_KIND / SWB_EL_FRAC in k_tma_common.cuh) were measured and reverted, see profiles/el_policy_r02.txt.
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for lib in "" el05 elnorm; do
    if [ -n "$lib" ]; then export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so; else unset SWB_LIB; fi
    timeout 300 python scripts/probe_k1perf.py 256:4 256:8 256:16 512:8 512:16
  done
done

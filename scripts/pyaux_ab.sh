#!/bin/bash
# SO 16 pencil: P_y in a fourth aux-ring slot (SWB_PY_AUX=1, default) vs its own 2-stage ring (pyold, a -DSWB_PY_AUX=0 build: build.py --variant pyold -DSWB_PY_AUX=0).
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for lib in "" pyold; do
    if [ -n "$lib" ]; then export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so; else unset SWB_LIB; fi
    timeout 300 python scripts/probe_k1perf.py 256:16 384:16
    SWB_YW=1 TAG="${lib:-libswb.so} YW=1" timeout 300 python scripts/probe_k1perf.py 512:16
  done
done

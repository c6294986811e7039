#!/bin/bash
# SO 8 y-pencil variant (28 rows + pencil = 16 warps, P_y through the aux ring), forced with SWB_YW=1, split point
# k >= 3 (default build), k >= 2 / k >= 4 (variant builds k4_2 / k4_4), against the 15-warp default.
cd "$(dirname "$0")/.."
for pass in 1 2; do
  unset SWB_LIB
  TAG=default timeout 300 python scripts/probe_k1perf.py 256:8 512:8
  SWB_YW=1 TAG="YW1 k>=3" timeout 300 python scripts/probe_k1perf.py 256:8 512:8
  for v in k4_2 k4_4; do
    SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$v.so SWB_YW=1 TAG="YW1 $v" timeout 300 python scripts/probe_k1perf.py 256:8 512:8
  done
done

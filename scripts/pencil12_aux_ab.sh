#!/bin/bash
# SO 12 pencil variant with P_y through the aux ring (28 rows + pencil warp = 16 warps, 128 registers), forced
# with SWB_YW=1 (queue unroll 2 and 4), against the 15-warp default.
cd "$(dirname "$0")/.."
for pass in 1 2; do
  TAG=default timeout 300 python scripts/probe_k1perf.py 256:12 384:12 512:12
  SWB_YW=1 SWB_UNR=2 TAG="YW1 UNR2" timeout 300 python scripts/probe_k1perf.py 256:12 384:12 512:12
  SWB_YW=1 SWB_UNR=4 TAG="YW1 UNR4" timeout 300 python scripts/probe_k1perf.py 256:12 384:12 512:12
done

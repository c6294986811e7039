#!/bin/bash
# SO 12 pencil variant queue unroll (UNR 1 / 2 / 3) with P_y through the aux ring (SWB_UNR forces the variant).
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for u in 1 2 3; do
    SWB_YW=1 SWB_T1=28 SWB_UNR=$u TAG="UNR $u" timeout 300 python scripts/probe_k1perf.py 256:12 384:12 512:12
  done
done

#!/bin/bash
# SO 16 pencil variant queue unroll (UNR 4 / 6 / 8) with P_y through the aux ring (SWB_UNR forces the variant).
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for u in ${UNRS:-4 6 8}; do
    SWB_YW=1 SWB_T1=20 SWB_UNR=$u TAG="UNR $u" timeout 300 python scripts/probe_k1perf.py 256:16 384:16 512:16
  done
done

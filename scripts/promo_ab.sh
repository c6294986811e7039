#!/bin/bash
# TMA L2 promotion of the u-box maps and the aux-tile maps (SWB_PROMO_U / SWB_PROMO_A), aligned z tiles.
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for pu in 256 128 0; do
    for pa in 256 128 0; do
      SWB_PROMO_U=$pu SWB_PROMO_A=$pa TAG="u$pu a$pa" timeout 300 python scripts/probe_k1perf.py 256:8 256:16 512:8
    done
  done
done

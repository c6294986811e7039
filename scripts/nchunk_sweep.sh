#!/bin/bash
# dim-0 chunk count sweep (SWB_NCHUNK) for K1 at 256^3 (development).
for so in 12 16; do for nc in 2 3 4 5 6 8 10 12; do
  echo "SO=$so NC=$nc $(SWB_NCHUNK=$nc timeout 60 python scripts/probe_perf.py factorised $so 256 200 2>&1 | tail -1)"
done; done

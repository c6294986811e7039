#!/bin/bash
# Env-selected K1 variants at 256^3 (development sweep; not the bench).
for so in 12 16; do
  for su in 10 11 14; do
    for unr in 2 4; do
      echo "SO=$so SU=$su UNR=$unr: $(SWB_SU=$su SWB_UNR=$unr timeout 120 python scripts/probe_perf.py factorised $so 256 200 2>&1 | tail -1)"
    done
  done
done

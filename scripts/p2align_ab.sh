#!/bin/bash
# Row pitch rounded to 64 floats vs 32 (SWB_P2ALIGN, a measured-and-reverted switch in runtime.cu): grids whose n2 is an odd multiple of 32.
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for pa in 32 64; do
    SWB_P2ALIGN=$pa TAG=p2align$pa timeout 300 python scripts/probe_k1perf.py 288:8 288:12 224:8 352:8 256:8
  done
done

#!/bin/bash
# SO 8 register queue: rotated by renaming (default, SWB_UNROLL_MAXH=4) vs shifted every UNR planes
# (variant build shq8: -DSWB_UNROLL_MAXH=3), pencil variant and plain.
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for lib in "" shq8; do
    if [ -n "$lib" ]; then export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so; else unset SWB_LIB; fi
    TAG="${lib:-rotate}" timeout 300 python scripts/probe_k1perf.py 256:8 512:8
    for u in 2 3 4; do
      SWB_UNR=$u TAG="${lib:-rotate} UNR $u" timeout 300 python scripts/probe_k1perf.py 256:8
    done
  done
done
